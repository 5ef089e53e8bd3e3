"""Model of the stream kernel's mbarrier protocol (biqgemm_stream.cu), run
under random schedules to search for deadlocks and protocol violations
(over-arrival, a waiter fooled by parity aliasing).  Every role is a
generator yielding ("wait", bar, parity) or ("arrive", bar, count); the
model mirrors the kernel's loops, barrier counts and parities.

    python tools/stream_protocol_sim.py            # sweep of shapes
Also used by tests/test_stream_protocol.py (CPU).
"""
from __future__ import annotations

import random
import sys


class Bar:
    def __init__(self, count):
        self.count = count
        self.pending = count
        self.phase = 0  # completed phases

    def arrive(self, cnt):
        if cnt > self.pending:
            raise AssertionError(f"over-arrival ({cnt} > {self.pending})")
        self.pending -= cnt
        if self.pending == 0:
            self.phase += 1
            self.pending = self.count

    def done(self, parity):
        return (self.phase & 1) != parity


def make(ncalls, U, ups, nst, nc, nlb, nab=2, nbuild=4, stagger=True):
    """Roles and barriers of biqgemm_stream_kernel: key warp lanes (one ring
    slot each, ungated, publishing issued[]), x loader (4 buffers), alpha
    loader (nab buffers), nbuild LUT builders (nlb buffers), nc gather warps
    (continuous unit assignment, call-aligned stages, count-completing
    arrival on a partial stage).  stagger: the kernel's ring start -- lane 0
    issues stage 0 alone, every issuing lane waits for its landing, then a
    __syncwarp of the issuing lanes (psync) before lane 0 may refill slot 0."""
    spc = (U + ups - 1) // ups
    B = {}
    for i in range(nst):
        B[("full", i)] = Bar(1)
        B[("empty", i)] = Bar(ups)
    for i in range(4):
        B[("xfull", i)] = Bar(1)
        B[("xempty", i)] = Bar(nbuild)
        B[("lfull", i)] = Bar(nbuild)
        B[("ldone", i)] = Bar(nc)
        B[("afull", i)] = Bar(1)
        B[("adone", i)] = Bar(nc)

    B[("psync",)] = Bar(nst)

    def producer(L):
        s = L
        if stagger and ncalls * spc > 1:
            if L == 0:
                yield ("set", ("issued", 0), 1)
                yield ("arrive", ("full", 0), 1)
            yield ("wait", ("full", 0), 0, 0)
            yield ("arrive", ("psync",), 1)
            yield ("wait", ("psync",), 0, 0)
            if L == 0:
                s = nst
        while s < ncalls * spc:
            rnd = s // nst
            if rnd > 0:
                yield ("wait", ("empty", L), (rnd - 1) & 1, rnd - 1)
            yield ("set", ("issued", L), rnd + 1)   # published after expect_tx
            yield ("arrive", ("full", L), 1)        # the copy lands (any time later)
            s += nst

    def xloader():
        for c in range(ncalls):
            if c >= 4:
                yield ("wait", ("xempty", c & 3), ((c >> 2) - 1) & 1, (c >> 2) - 1)
            yield ("arrive", ("xfull", c & 3), 1)

    def aloader():
        for c in range(ncalls):
            if c >= nab:
                yield ("wait", ("adone", c % nab), (c // nab - 1) & 1, c // nab - 1)
            yield ("arrive", ("afull", c % nab), 1)

    def builder(q):
        for c in range(ncalls):
            yield ("wait", ("xfull", c & 3), (c >> 2) & 1, c >> 2)
            if c >= nlb:
                yield ("wait", ("ldone", c % nlb), (c // nlb - 1) & 1, c // nlb - 1)
            yield ("arrive", ("xempty", c & 3), 1)
            yield ("arrive", ("lfull", c % nlb), 1)

    def consumer(w):
        gu = w
        for c in range(ncalls):
            yield ("wait", ("lfull", c % nlb), (c // nlb) & 1, c // nlb)
            yield ("wait", ("afull", c % nab), (c // nab) & 1, c // nab)
            while gu < (c + 1) * U:
                k = gu - c * U
                sj, pos = divmod(k, ups)
                st = c * spc + sj
                yield ("atleast", ("issued", st % nst), st // nst + 1)
                yield ("wait", ("full", st % nst), (st // nst) & 1, st // nst)
                nin = min(ups, U - sj * ups)
                yield ("arrive", ("empty", st % nst), ups - nin + 1 if pos == nin - 1 else 1)  # x32 lanes in the kernel
                gu += nc
            yield ("arrive", ("ldone", c % nlb), 1)
            yield ("arrive", ("adone", c % nab), 1)

    procs = [producer(L) for L in range(nst)]
    procs += [xloader(), aloader()]
    procs += [builder(q) for q in range(nbuild)]
    procs += [consumer(w) for w in range(nc)]
    return B, procs


def run(ncalls, U, ups, nst, nc, nlb, nab=2, seed=0, stagger=True):
    """Returns None if every role finishes, else a description of the failure."""
    rng = random.Random(seed)
    B, procs = make(ncalls, U, ups, nst, nc, nlb, nab, stagger=stagger)
    cur = [next(p, None) for p in procs]
    cnt = {}
    while True:
        live = [i for i, op in enumerate(cur) if op is not None]
        if not live:
            return None
        ready = []
        for i in live:
            op = cur[i]
            if op[0] in ("arrive", "set"):
                ready.append(i)
            elif op[0] == "atleast":
                if cnt.get(op[1], 0) >= op[2]:
                    ready.append(i)
            else:
                bar = B[op[1]]
                if bar.done(op[2]):
                    # parity aliasing: the barrier must have completed exactly the
                    # phase the waiter means (phase index op[3]), not two later
                    if bar.phase - 1 != op[3] and bar.phase - 1 > op[3]:
                        if (bar.phase - 1 - op[3]) % 2 == 0 and bar.phase - 1 - op[3] >= 2:
                            return f"parity alias on {op[1]}: wanted phase {op[3]}, barrier at {bar.phase - 1}"
                    ready.append(i)
                elif bar.phase > op[3] + 1:
                    return f"parity alias (blocked) on {op[1]}: wanted phase {op[3]}, barrier completed {bar.phase}"
        if not ready:
            waits = {str(cur[i][1]) for i in live}
            return f"deadlock: {len(live)} roles blocked on {sorted(waits)[:6]}"
        i = rng.choice(ready)
        op = cur[i]
        if op[0] == "set":
            cnt[op[1]] = op[2]
        elif op[0] == "arrive":
            try:
                B[op[1]].arrive(op[2])
            except AssertionError as e:
                return f"{op[1]}: {e}"
        cur[i] = next(procs[i], None)


def sweep(seeds=3, verbose=False):
    bad = []
    for U in (1, 2, 3, 5, 14, 15, 18, 19, 40, 57):
        for ups in (3, 4, 6, 12):
            for nst in (2, 3, 6, 9, 12):
                for nlb in (2, 4):
                    for nab in (2, 4):
                        for ncalls in (1, 2, 3, 7, 12):
                            for sd in range(seeds):
                                r = run(ncalls, U, ups, nst, 18, nlb, nab, seed=sd)
                                if r:
                                    bad.append((U, ups, nst, nlb, nab, ncalls, sd, r))
                                    if verbose:
                                        print(bad[-1])
                                    break
    return bad


if __name__ == "__main__":
    b = sweep(seeds=int(sys.argv[1]) if len(sys.argv) > 1 else 3, verbose=True)
    print("failures:", len(b))
