"""CPU tests of the C-ABI library: it loads, exports every declared symbol,
its host-side logic matches the reference, and compute entry points fail
loudly (no CPU fallback) when no device is present."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "bqg_capi.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bqg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2005_09904_b200 import _capi

    names = declared_symbols()
    assert len(names) >= 30
    for name in names:
        assert hasattr(_capi.lib, name), name
        assert name in _capi.SIGNATURES, f"{name} not bound in _capi.SIGNATURES"
    assert _capi.lib.bqg_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess

    from paper_2005_09904_b200 import _capi

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_rng_matches_reference(bq, ref):
    for seed in (0, 1, 0x5EED, 2**63 + 5):
        assert np.array_equal(bq.random_uniform(7, 13, seed), ref.random_uniform(7, 13, seed))
        assert np.array_equal(bq.random_normal(13, 3, seed), ref.random_normal(13, 3, seed))
        assert np.array_equal(bq.random_uniform(3, 5, seed, -2.0, 3.0), ref.random_uniform(3, 5, seed, -2.0, 3.0))


def test_plan_tiles_matches_reference(bq, port):
    rng = np.random.default_rng(5)
    for _ in range(200):
        m, groups, b, mu = (int(rng.integers(1, 5000)), int(rng.integers(1, 600)), int(rng.integers(1, 300)),
                            int(rng.integers(1, 12)))
        budget = int(rng.integers(1, 1 << 20))
        try:
            want = port.plan_tiles(m, groups, b, mu, budget, 4)
        except ValueError:
            with pytest.raises(ValueError):
                bq.plan_tiles(m, groups, b, mu, budget, 4)
            continue
        t = bq.plan_tiles(m, groups, b, mu, budget, 4)
        assert (t.t_w, t.t_h) == want


def test_footprint_table_ii(bq):  # acceptance criterion 5, test_model_io.cpp:82-97
    want = {32: 1.049, 8: 0.262, 6: 0.197, 4: 0.131, 3: 0.098, 2: 0.066}
    for bits, mb in want.items():
        assert round(bq.footprint(512, 512, bits).weight_mb(), 3) == mb
    assert bq.footprint(512, 512, 4).weight_bytes == 131072
    f = bq.footprint(512, 512, 4, 18)
    assert round(f.activation_mb(), 3) == 0.037 and round(f.output_mb(), 3) == 0.037
    with pytest.raises(ValueError):
        bq.footprint(1, 1, 0)


def test_footprint_matches_reference(bq, ref):
    for m, n, bits, batch in [(512, 512, 3, 18), (7, 9, 5, 1), (4096, 4096, 2, 32)]:
        f = bq.footprint(m, n, bits, batch)
        assert [f.weight_bytes, f.activation_bytes, f.output_bytes, f.alpha_bytes] == ref.footprint(m, n, bits, batch)


def test_counter_laws(bq, port):  # acceptance criterion 3
    rng = np.random.default_rng(0x5EED)
    for _ in range(20):
        m, n, b = int(rng.integers(1, 65)), int(rng.integers(1, 101)), int(rng.integers(1, 9))
        mu, beta = int(rng.integers(1, 9)), int(rng.integers(1, 4))
        G = (n + mu - 1) // mu
        c = bq.op_counters(m, n, b, beta, mu)
        assert c["lut_build_ops"] == ((1 << mu) + mu - 1) * G * b
        assert c["lookups"] == m * G * b * beta == c["accumulate_ops"]
    assert bq.op_counters(512, 512, 18, 1, 8)["lookups"] == 589824


def test_bqgm_roundtrip_vs_reference(bq, ref):
    rng = np.random.default_rng(0x5EED)
    for _ in range(25):  # test_model_io.cpp:28-45
        m, n, beta, mu = int(rng.integers(1, 13)), int(rng.integers(1, 25)), int(rng.integers(1, 4)), int(
            rng.integers(1, 13))
        w = ref.random_uniform(m, n, int(rng.integers(0, 2**62)))
        data = ref.save_bqgm(w, beta, mu)
        mm, nn, bb, uu, alpha, keys = bq.parse_bqgm(data)
        st, rm, rn, rb, ru, rkeys, ralpha = ref.load_bqgm(data)
        assert st == 0 and (mm, nn, bb, uu) == (rm, rn, rb, ru)
        assert np.array_equal(keys.astype(np.uint32), rkeys) and np.array_equal(alpha, ralpha)
        assert bq.serialize_bqgm(keys, alpha, mm, nn, bb, uu) == data  # byte-identical save()


def test_bqgm_typed_errors(bq, ref):  # test_model_io.cpp:56-78
    from paper_2005_09904_b200 import _capi

    w = ref.random_uniform(4, 8, 6)
    good = bytearray(ref.save_bqgm(w, 1, 3))
    cases = []
    bad = bytearray(good)
    bad[0] = ord("X")
    cases.append((bytes(bad), _capi.BadMagicError, 2))
    bad = bytearray(good)
    bad[4] = 99
    cases.append((bytes(bad), _capi.BadVersionError, 3))
    cases.append((bytes(good[: len(good) // 2]), _capi.TruncatedError, 4))
    bad = bytearray(good)
    bad[-1] = 0xFF
    cases.append((bytes(bad), _capi.RangeError, 5))
    cases.append((bytes(good) + b"\0", _capi.FormatError, 6))
    cases.append((bytes(good[:2]), _capi.TruncatedError, 4))
    hdr0 = bytearray(good)
    hdr0[6:10] = b"\0\0\0\0"  # m = 0
    cases.append((bytes(hdr0), _capi.RangeError, 5))
    for data, exc, ref_status in cases:
        assert ref.load_bqgm(data)[0] == ref_status
        with pytest.raises(exc):
            bq.parse_bqgm(data)


def test_no_cpu_fallback_without_device(bq):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2005_09904_b200 import _capi

    with pytest.raises(_capi.NoDeviceError):
        bq.PackedLinear.from_weights(np.ones((4, 8), np.float32), 1, 4)
    st = _capi.lib.bqg_quantize_greedy_f32(1, 4, 8, 1, 1, 1, None)
    assert st == _capi.BQG_ERR_NO_DEVICE


def test_validation_matches_reference_exceptions(bq):
    from paper_2005_09904_b200 import _capi

    lib = _capi.lib
    assert lib.bqg_pack_keys(1, 4, 4, 0, 1, None) == _capi.BQG_ERR_INVALID_ARGUMENT  # mu range
    assert lib.bqg_pack_keys(1, 4, 4, 17, 1, None) == _capi.BQG_ERR_INVALID_ARGUMENT
    assert lib.bqg_quantize_greedy_f32(1, 4, 8, 0, 1, 1, None) == _capi.BQG_ERR_INVALID_ARGUMENT  # beta=0
    # key matrix too narrow for x (kernel.hpp:132-134): n=8, mu=4 -> G*mu=8 < 16 rows
    assert lib.bqg_biqgemm_f32(1, 1, 1, 16, 1, 4, 8, 1, 1, 4, 1, 1 << 20, 0, None) == _capi.BQG_ERR_INVALID_ARGUMENT
    with pytest.raises(_capi.InvalidArgument):
        bq.plan_tiles(1024, 128, 64, 8, 1024, 4)
