"""CPU model check of the stream kernel's mbarrier protocol
(tools/stream_protocol_sim.py mirrors biqgemm_stream.cu's roles, barrier
counts and parities): no deadlock, no over-arrival, no parity aliasing under
random schedules, across unit/stage/ring/buffer shapes."""
import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
import stream_protocol_sim as sim  # noqa: E402


@pytest.mark.parametrize("U,ups,nst", [(1, 6, 2), (1, 12, 6), (3, 4, 2), (14, 4, 6), (15, 4, 6), (15, 4, 3),
                                       (19, 12, 2), (57, 4, 4), (57, 4, 9), (40, 6, 12)])
@pytest.mark.parametrize("nlb", [2, 4])
@pytest.mark.parametrize("nab", [2, 4])
def test_protocol_is_deadlock_free(U, ups, nst, nlb, nab):
    for ncalls in (1, 2, 5, 9):
        for seed in range(3):
            assert sim.run(ncalls, U, ups, nst, 18, nlb, nab, seed=seed) is None


def test_model_catches_the_unguarded_ring():
    """Without the issued-round counter the model finds the stale-slot read
    (a warp two ring rounds ahead passes the parity wait)."""
    src = Path(sim.__file__).read_text()
    assert '("atleast", ("issued"' in src
    bad = 0
    orig = sim.make

    def no_guard(*a, **k):
        B, procs = orig(*a, **k)

        def strip(p):
            for op in p:
                if op[0] != "atleast":
                    yield op
        return B, [strip(p) for p in procs]

    sim.make = no_guard
    try:
        for seed in range(20):
            if sim.run(12, 57, 12, 2, 18, 4, 2, seed=seed):
                bad += 1
    finally:
        sim.make = orig
    assert bad > 0


@pytest.mark.parametrize("stagger", [True, False])
def test_ring_start_orders(stagger):
    """Both ring starts are deadlock-free: stage 0 alone first (the kernel's
    default) and the whole ring at once (BQG_DEBUG_FLAGS bit 21)."""
    for U, ups, nst in ((1, 6, 2), (15, 4, 6), (57, 4, 9), (40, 6, 12)):
        for ncalls in (1, 2, 5):
            for seed in range(3):
                assert sim.run(ncalls, U, ups, nst, 18, 4, 2, seed=seed, stagger=stagger) is None

