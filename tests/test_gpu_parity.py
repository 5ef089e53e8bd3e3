"""Parity of the CUDA path (through the C ABI) against the oracle.

Bars (BASELINE.json north_star):
  - sign planes, alpha, keys, tiled keys, LUT indices: bit-exact;
  - fast-path LUT (fp32): bit-exact with the DP evaluated in fp32 (port);
  - exact-path LUT and y (fp64): bit-exact with the reference;
  - fast-path y: ||y - y_ref||_F / ||y_ref||_F <= 1e-5 and
    max|y - y_ref| <= 1e-5 * max|y_ref| (y_ref = the reference's own
    biqgemm, fp64 accumulation).
"""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
TOL = 1e-5


def assert_close(y, y_ref, tol=TOL):
    y = np.asarray(y, np.float64)
    y_ref = np.asarray(y_ref, np.float64)
    nrm = np.linalg.norm(y_ref)
    rel = np.linalg.norm(y - y_ref) / nrm if nrm > 0 else np.linalg.norm(y - y_ref)
    mx = np.max(np.abs(y_ref)) if y_ref.size else 0.0
    assert rel <= tol, f"relative Frobenius {rel:.3e} > {tol}"
    assert np.max(np.abs(y - y_ref)) <= tol * max(mx, 1e-30), "max abs error"


def cases():
    d = np.load(GOLD / "cases.npz")
    for i in range(int(d["count"][0])):
        yield {k[len(f"c{i}_"):]: d[k] for k in d.files if k.startswith(f"c{i}_")}


def tile_numpy(keys, mu):
    """The tiled layout of kernels.h restated in numpy."""
    beta, m, G = keys.shape
    MT, NB = (m + 31) // 32, (G + 31) // 32
    kp = np.zeros((beta, MT * 32, NB * 32), np.uint8)
    kp[:, :m, :G] = keys
    out = np.zeros((NB, MT, beta, 2, 32, 16), np.uint8)
    for l in range(32):
        for j in range(32):
            gl = (l + j) % 32
            # kp[i, t*32 + l, gb*32 + gl] for all (i, t, gb)
            out[:, :, :, j >> 4, l, j & 15] = kp[:, l::32, gl::32].transpose(2, 1, 0)
    return out.reshape(-1)


# ------------------------------------------------------------------ producers


def test_quantize_pack_bit_exact_on_fixtures(bq, cuda):
    import torch

    for c in cases():
        m, n, b, beta, mu, wseed, xseed = (int(v) for v in c["dims"])
        w = bq.random_uniform(m, n, wseed)
        planes, alpha = bq.quantize_greedy(torch.from_numpy(w), beta)
        assert np.array_equal(planes.cpu().numpy().view(np.uint32), c["planes"])
        assert np.array_equal(alpha.cpu().numpy(), c["alpha"])
        for i in range(beta):
            keys = bq.pack_keys(planes[i], n, mu).cpu().numpy()
            keys = keys.view(np.uint16) if mu > 8 else keys
            assert np.array_equal(keys, c["keys"][i].astype(keys.dtype))


def test_layer_from_weights_matches_reference(bq, cuda, port):
    rng = np.random.default_rng(11)
    for _ in range(10):
        m, n, beta, mu = int(rng.integers(1, 200)), int(rng.integers(1, 300)), int(rng.integers(1, 4)), int(
            rng.integers(1, 17))
        w = bq.random_uniform(m, n, int(rng.integers(0, 2**62)))
        layer = bq.PackedLinear.from_weights(w, beta, mu)
        keys, alpha, planes = layer.export(planes=True)
        p_planes, p_alpha = port.quantize_greedy(w, beta)
        assert np.array_equal(planes, p_planes) and np.array_equal(alpha, p_alpha)
        p_keys = np.stack([port.pack_keys(p_planes[i], n, mu) for i in range(beta)])
        assert np.array_equal(keys.astype(np.uint32), p_keys)
        layer.close()


def test_tile_layout(bq, cuda):
    import torch

    rng = np.random.default_rng(2)
    for m, G, beta in [(1, 1, 1), (31, 33, 2), (64, 64, 3), (100, 70, 1), (4096, 512, 1)]:
        keys = rng.integers(0, 256, size=(beta, m, G), dtype=np.uint8)
        tiled = bq.tile_keys(torch.from_numpy(keys).cuda(), G * 8, 8).cpu().numpy()
        assert np.array_equal(tiled, tile_numpy(keys, 8))


def test_config_c2_keys_sha(bq, cuda):
    import hashlib

    meta = json.loads((GOLD / "configs.json").read_text())["C2"]
    w = bq.random_uniform(4096, 4096, 0x5EED)
    layer = bq.PackedLinear.from_weights(w, 3, 8)
    keys, alpha = layer.export()
    assert hashlib.sha256(keys.tobytes()).hexdigest() == meta["keys_sha"]
    assert hashlib.sha256(alpha.tobytes()).hexdigest() == meta["alpha_sha"]


# ----------------------------------------------------------------------- LUT


def test_fast_lut_bit_exact_with_fp32_dp(bq, port, cuda):
    rng = np.random.default_rng(3)
    for mu in range(1, 9):
        for b in (1, 2, 3, 5):
            x_rows = int(rng.integers(1, 200))
            x = rng.standard_normal((x_rows, b)).astype(np.float32) * 3
            G = (x_rows + mu - 1) // mu + int(rng.integers(0, 3))  # includes all-zero padded groups
            g0 = int(rng.integers(0, 3))
            count = max(1, G - g0)
            for layout in (bq.TableMajor, bq.KeyMajor):
                got, ops = bq.build_lut_block(x, g0, count, mu, layout, "f32")
                want, wops = port.build_lut_block(x, g0, count, mu, key_major=layout == bq.KeyMajor, dtype=np.float32)
                assert np.array_equal(got.cpu().numpy(), want), (mu, b, layout)
                assert ops == wops
                tbl = got.cpu().numpy().reshape(count, b, 1 << mu) if layout == bq.TableMajor else None
                if tbl is not None:  # complement negation is bitwise
                    half = 1 << (mu - 1)
                    assert np.array_equal(tbl[:, :, ::-1][:, :, :half], -tbl[:, :, :half])


def test_exact_lut_bit_exact_with_reference(bq, cuda):
    for c in cases():
        if "lut_t" not in c:
            continue
        m, n, b, beta, mu, wseed, xseed = (int(v) for v in c["dims"])
        x = bq.random_normal(n, b, xseed)
        G = (n + mu - 1) // mu
        got_t, _ = bq.build_lut_block(x, 0, G, mu, bq.TableMajor, "f64")
        got_k, _ = bq.build_lut_block(x, 0, G, mu, bq.KeyMajor, "f64")
        assert np.array_equal(got_t.cpu().numpy(), c["lut_t"])
        assert np.array_equal(got_k.cpu().numpy(), c["lut_k"])


def test_exact_lut_large_mu_vs_reference(bq, ref, cuda):
    rng = np.random.default_rng(4)
    for mu in (9, 12, 16):
        x = rng.standard_normal((40, 2)).astype(np.float32)
        G = (40 + mu - 1) // mu
        got, _ = bq.build_lut_block(x, 0, G, mu, bq.TableMajor, "f64")
        want, _ = ref.build_lut_block(x, 0, G, mu)
        assert np.array_equal(got.cpu().numpy(), want)


# -------------------------------------------------------------------- BiQGEMM


def test_fixtures_fast_and_exact(bq, cuda):
    for c in cases():
        m, n, b, beta, mu, wseed, xseed = (int(v) for v in c["dims"])
        x = bq.random_normal(n, b, xseed)
        keys = c["keys"]
        layer = bq.PackedLinear.from_keys(keys, c["alpha"], n, mu)
        y_exact = layer.forward(x, exact=True)
        assert np.array_equal(y_exact, c["y"]), f"exact path not bit-identical (mu={mu})"
        assert_close(layer.forward(x), c["y"])  # mu > 8: the re-keyed mu = 8 fast path
        plane = bq.PackedLinear.from_keys(keys[:1], None, n, mu)
        assert np.array_equal(plane.forward(x, exact=True), c["yplane"])
        assert_close(plane.forward(x), c["yplane"])
        layer.close()
        plane.close()


def test_acceptance_style_random_cases(bq, port, cuda):
    """acceptance_test.cpp:45-89 generator (criterion 1) through the GPU path:
    fp32 vs dequantized dense <= 1e-4 (the reference's own bar) and vs the
    reference's own BiQGEMM <= 1e-5."""
    rng = np.random.Generator(np.random.PCG64(0x5EED))
    for _ in range(200):
        m, n, b = int(rng.integers(1, 65)), int(rng.integers(1, 65)), int(rng.integers(1, 9))
        mu = int(rng.choice([1, 2, 4, 8]))
        beta = int(rng.integers(1, 4))
        w = bq.random_uniform(m, n, int(rng.integers(0, 2**62)))
        x = bq.random_normal(n, b, int(rng.integers(0, 2**62)))
        layer = bq.PackedLinear.from_weights(w, beta, mu)
        keys, alpha, planes = layer.export(planes=True)
        y = layer.forward(x)
        y_ref, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, mu, x)
        assert_close(y, y_ref)
        dense = port.gemm_dense(port.dequantize(planes, alpha, n), x)
        assert port.rel_frobenius(y, dense) <= 1e-4
        layer.close()


@pytest.mark.parametrize("m,n,b,beta,mu", [
    (1, 1, 1, 1, 8), (1, 8, 1, 1, 8), (33, 7, 1, 2, 3), (100, 300, 1, 3, 8), (100, 300, 2, 3, 8),
    (100, 300, 3, 2, 8), (70, 257, 4, 1, 8), (257, 1000, 5, 2, 7), (64, 2048, 8, 3, 8), (96, 1024, 32, 2, 8),
    (1024, 1024, 1, 1, 8), (2000, 4100, 1, 3, 8), (300, 600, 17, 2, 6), (40, 90, 6, 3, 5),
])
def test_shapes_vs_port(bq, port, cuda, m, n, b, beta, mu):
    w = bq.random_uniform(m, n, 1000 + m)
    x = bq.random_normal(n, b, 2000 + n)
    layer = bq.PackedLinear.from_weights(w, beta, mu)
    keys, alpha = layer.export()
    y_ref, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, mu, x)
    y = layer.forward(x)
    assert_close(y, y_ref)
    assert np.array_equal(layer.forward(x), y)  # deterministic
    assert np.array_equal(layer.forward(x, exact=True), y_ref)


def test_short_x_is_zero_padded(bq, port, cuda):
    w = bq.random_uniform(50, 100, 5)
    layer = bq.PackedLinear.from_weights(w, 2, 8)  # G = 13 -> G*mu = 104
    keys, alpha = layer.export()
    for rows in (1, 37, 100, 104):
        x = bq.random_normal(rows, 3, rows)
        y_ref, _ = port.biqgemm(keys.astype(np.uint32), alpha, 100, 8, x)
        assert_close(layer.forward(x), y_ref)
    from paper_2005_09904_b200 import _capi

    with pytest.raises(_capi.InvalidArgument):
        layer.forward(np.zeros((105, 1), np.float32))


def test_row_sharding_is_bitwise_invariant(bq, cuda):
    """Row-sharded layers (the multi-GPU decomposition, shard boundaries on
    32-row tiles) reproduce the full y bitwise."""
    w = bq.random_uniform(1000, 777, 9)
    x = bq.random_normal(777, 3, 10)
    full = bq.PackedLinear.from_weights(w, 3, 8)
    keys, alpha = full.export()
    y = full.forward(x)
    y1 = full.forward(x[:, :1].copy())
    for k in (2, 3, 8):
        bounds = [min(1000, 32 * ((1000 * i // k + 31) // 32)) for i in range(k + 1)]
        parts, parts1 = [], []
        for a, z in zip(bounds[:-1], bounds[1:]):
            shard = bq.PackedLinear.from_keys(keys[:, a:z], alpha[:, a:z], 777, 8)
            parts.append(shard.forward(x))
            parts1.append(shard.forward(x[:, :1].copy()))
            shard.close()
        assert np.array_equal(np.concatenate(parts), y)
        assert np.array_equal(np.concatenate(parts1), y1)


def test_bqgm_load_forward(bq, ref, cuda):
    w = ref.random_uniform(300, 500, 77)
    data = ref.save_bqgm(w, 2, 8)
    layer = bq.PackedLinear.load(data)
    _, _, _, _, rkeys, ralpha = ref.load_bqgm(data)[1:]
    x = ref.random_normal(500, 4, 78)
    y_ref, _ = ref.biqgemm(rkeys, ralpha, 500, 8, x)
    assert np.array_equal(layer.forward(x, exact=True), y_ref)
    assert_close(layer.forward(x), y_ref)
    layer12 = bq.PackedLinear.load(ref.save_bqgm(w, 2, 12))
    _, _, _, _, _, k12, a12 = ref.load_bqgm(ref.save_bqgm(w, 2, 12))
    y12, _ = ref.biqgemm(k12, a12, 500, 12, x)
    assert np.array_equal(layer12.forward(x, exact=True), y12)
    assert_close(layer12.forward(x), y12)  # the re-keyed mu = 8 fast path


def test_large_mu_random_sweep(cuda):
    """tools/rand_large_mu.py: random (m, n, beta, mu 9..16, b, x rows up to
    G*mu) through the re-keyed fast path against the C oracle (rel-Frobenius
    and max-abs <= 1e-5), grouped host calls bitwise equal to single calls."""
    import subprocess
    import sys

    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "tools" / "rand_large_mu.py"), "40"], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "cases ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("m,n,beta,mu", [(300, 500, 2, 12), (1000, 777, 3, 10), (64, 4096, 1, 9), (96, 1000, 2, 16),
                                         (4096, 4096, 3, 10), (33, 13, 2, 11),
                                         # mu < 8 layers are re-keyed to mu = 8 too
                                         (300, 500, 2, 4), (1000, 777, 3, 6), (64, 4096, 1, 1), (96, 1000, 2, 7),
                                         (4096, 4096, 3, 5), (33, 13, 2, 3), (2000, 3000, 4, 2)])
def test_large_mu_fast_path_rekeyed(bq, port, cuda, m, n, beta, mu):
    """mu > 8 on the fast path: the sign bits re-keyed to mu = 8 over
    8*ceil(G*mu/8) columns run the mu <= 8 kernels.  y within the fp32
    contract of the reference's mu-bit result for every x length the mu-keys
    accept -- x shorter than n, x = n, and x = G*mu rows (past n: the pad
    bits' sign); the re-keyed bytes are the mu = 8 packing of the same
    bits."""
    import ctypes as C

    import torch

    w = bq.random_uniform(m, n, 11 + mu)
    layer = bq.PackedLinear.from_weights(w, beta, mu)
    keys, alpha = layer.export()
    G = (n + mu - 1) // mu
    n8, mu8 = C.c_size_t(), C.c_uint()
    bq.check(bq.lib.bqg_layer_fast_shape(layer._h, C.byref(n8), C.byref(mu8)))
    assert (n8.value, mu8.value) == (8 * ((G * mu + 7) // 8), 8)
    # the re-keyed bytes: the same sign bits packed 8 per byte
    bits = ((keys.astype(np.uint32)[..., None] >> np.arange(mu, dtype=np.uint32)) & 1).reshape(beta, m, G * mu)
    bits = np.concatenate([bits, np.zeros((beta, m, n8.value - G * mu), np.uint32)], axis=2)
    want8 = (bits.reshape(beta, m, -1, 8) << np.arange(8, dtype=np.uint32)).sum(-1).astype(np.uint8)
    kd = torch.from_numpy(keys.view(np.int16) if mu > 8 else keys).cuda()
    out = torch.empty((beta, m, n8.value // 8), dtype=torch.uint8, device="cuda")
    bq.check(bq.lib.bqg_rekey_mu8(kd.data_ptr(), m, n, beta, mu, out.data_ptr(), None))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want8)
    for rows, b in ((n, 1), (n, 3), (max(1, n // 2), 2), (G * mu, 1)):
        x = bq.random_normal(rows, b, 5 + rows)
        y_ref, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, mu, x)
        assert_close(layer.forward(x), y_ref)
        assert np.array_equal(layer.forward(x, exact=True), layer.forward(x, exact=True))
    # a group of such layers through the grouped host pipeline == one by one,
    # for x of n rows and of G*mu rows (the whole re-keyed width when it is
    # wider than 8*ceil(n/8))
    for rows in sorted({n, G * mu}):
        xs = np.stack([bq.random_normal(rows, 1, 40 + i) for i in range(6)])
        yg = bq.layers_forward([layer] * 6, xs)
        for i in range(6):
            assert np.array_equal(yg[i], layer.forward(xs[i]))
        y_ref, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, mu, xs[5])
        assert_close(yg[5], y_ref)
    layer.close()


def test_stats_counters_and_accumulation(bq, cuda):
    from paper_2005_09904_b200._capi import KernelStats

    layer = bq.PackedLinear.from_weights(bq.random_uniform(512, 512, 1), 1, 8)
    st = KernelStats()
    x = bq.random_normal(512, 18, 2)
    layer.forward(x, stats=st)
    assert st.lookups == 589824 and st.accumulate_ops == 589824
    assert st.lut_build_ops == (256 + 8 - 1) * 64 * 18
    layer.forward(x, stats=st)
    assert st.lookups == 2 * 589824  # accumulates like KernelStats (kernel.hpp:197-202)
    assert st.query_seconds > 0 and st.replace_seconds > 0


def test_fault_injection_is_detected(bq, port, cuda):
    """Mutation test (bench_cli --inject-pack-fault analogue): flipping one
    tiled key byte must break parity."""
    import torch

    m, n, beta, mu = 256, 512, 2, 8
    w = bq.random_uniform(m, n, 3)
    layer = bq.PackedLinear.from_weights(w, beta, mu)
    keys, alpha = layer.export()
    x = bq.random_normal(n, 1, 4)
    y_ref, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, mu, x)
    tiled = bq.tile_keys(torch.from_numpy(keys).cuda(), n, mu)
    a_d = torch.from_numpy(alpha).cuda()
    x_d = torch.from_numpy(x).cuda()
    y_d = torch.empty((m, 1), device="cuda")
    ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, 1, beta, mu)))
    bq.biqgemm_device(tiled, a_d, x_d, y_d, m, n, beta, mu, ws)
    assert_close(y_d.cpu().numpy(), y_ref)
    tiled[12345] ^= 0x5A
    bq.biqgemm_device(tiled, a_d, x_d, y_d, m, n, beta, mu, ws)
    with pytest.raises(AssertionError):
        assert_close(y_d.cpu().numpy(), y_ref)


def test_pdl_chain_and_graph(bq, port, cuda):
    """Back-to-back PDL launches on one stream (and inside a CUDA graph) keep
    stream semantics: a chain y1 = f(x), y2 = f(y1) matches the oracle."""
    import torch

    m = n = 2048
    layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, 21), 2, 8)
    keys, alpha = layer.export()
    x = bq.random_normal(n, 1, 22)
    xd = torch.from_numpy(x).cuda()
    y1 = torch.empty((m, 1), device="cuda")
    y2 = torch.empty((m, 1), device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        layer.forward_device(xd, y1, pdl=True)
        layer.forward_device(y1, y2, pdl=True)
    s.synchronize()
    r1, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, 8, x)
    r2, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, 8, y1.cpu().numpy())
    assert_close(y1.cpu().numpy(), r1)
    assert_close(y2.cpu().numpy(), r2)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        layer.forward_device(xd, y1, pdl=True)  # warm
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            layer.forward_device(xd, y1, pdl=True)
            layer.forward_device(y1, y2, pdl=True)
    y1.zero_()
    y2.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert_close(y1.cpu().numpy(), r1)
    assert_close(y2.cpu().numpy(), r2)


BASELINE_POINTS = ["C1", "C2", "C3"] + [f"C4b{b}" for b in (1, 2, 4, 8, 16, 32, 64, 128, 256)] + ["C5"]


@pytest.mark.parametrize("name", BASELINE_POINTS)
def test_baseline_configs(bq, cuda, name):
    """Every BASELINE config point on the bench_cli data (seeds 0x5EED /
    0x5EED+1, bench_cli.cpp:106-109) against the REFERENCE's own output
    (tests/golden/make_golden.py ran biqgemm::biqgemm, kernel.hpp:246-258):
      - the GPU quantize/pack reproduces the reference's keys and alpha (sha256);
      - the exact path reproduces the reference's y bit for bit (sha256 of the
        whole y, and its checksum);
      - the fast path meets the fp32 contract against that y (and the stored
        reference rows).
    C4 covers the whole batch sweep b = 1..256 (configs[3]); C5 is the
    multi-GPU config (65536 x 8192, q2, b8) computed whole on one GPU."""
    import hashlib

    meta = json.loads((GOLD / "configs.json").read_text())[name]
    m, n, beta, b = meta["m"], meta["n"], meta["beta"], meta["b"]
    layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, 0x5EED), beta, 8)
    keys, alpha = layer.export()
    assert hashlib.sha256(keys.astype(np.uint8).tobytes()).hexdigest() == meta["keys_sha"]
    assert hashlib.sha256(alpha.tobytes()).hexdigest() == meta["alpha_sha"]
    x = bq.random_normal(n, b, 0x5EED + 1)
    assert hashlib.sha256(x.tobytes()).hexdigest() == meta["x_sha"]
    y_exact = layer.forward(x, exact=True)
    assert float(np.sum(y_exact.astype(np.float64))) == meta["checksum"]
    assert hashlib.sha256(np.ascontiguousarray(y_exact).tobytes()).hexdigest() == meta["y_sha"]
    gold = np.load(GOLD / "configs.npz")
    if name + "_y" in gold.files:
        assert np.array_equal(y_exact, gold[name + "_y"])
    y = layer.forward(x)
    assert_close(y, y_exact)
    if name + "_ysample" in gold.files:
        ys = gold[name + "_ysample"]
        assert np.array_equal(y_exact[:: meta["sample_stride"]], ys)
        assert_close(y[:: meta["sample_stride"]], ys)
    layer.close()


@pytest.mark.parametrize("flags", ["8192", "128"])
def test_both_fast_forms(cuda, flags):
    """Force each fast-path form (single-kernel cluster / two-kernel) on
    assorted shapes in a subprocess (the form switch is read once per process)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, BQG_DEBUG_FLAGS=flags)
    r = subprocess.run([sys.executable, str(Path(__file__).parent / "forms_check.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_naive_builder_exact_path_vs_reference(bq, cuda):
    """KernelOptions::builder = Naive runs the exact path with naive fp64
    tables: y bit-identical to the reference run with LutBuilder::Naive
    (tests/golden/naive.npz), counters with the naive law, and a real
    build / query / replace phase split (kernel.hpp:156-159)."""
    from paper_2005_09904_b200._capi import LUT_NAIVE, KernelStats

    d = np.load(Path(__file__).resolve().parent / "golden" / "naive.npz")
    for i in range(int(d["count"][0])):
        c = {k[len(f"n{i}_"):]: d[k] for k in d.files if k.startswith(f"n{i}_")}
        m, n, b, beta, mu = (int(v) for v in c["dims"])
        keys = c["keys"].astype(np.uint16 if mu > 8 else np.uint8)
        layer = bq.PackedLinear.from_keys(keys, c["alpha"], n, mu)
        st = KernelStats()
        y = layer.forward(c["x"], stats=st, builder=LUT_NAIVE)
        assert np.array_equal(y, c["y_naive"]), f"case {i}"
        assert [st.lut_build_ops, st.lookups, st.accumulate_ops] == [int(v) for v in c["counters"]]
        assert st.build_seconds > 0 and st.query_seconds > 0 and st.replace_seconds > 0
        assert np.array_equal(layer.forward(c["x"], exact=True), c["y_dp"])  # the Dp builder, exact path
        layer.close()


def test_exact_ex_entry_phase_split(bq, cuda):
    """bqg_biqgemm_exact_ex_f32 on device buffers: builder choice and the
    event-timed phase split; the fast path reports its build inside query."""
    import ctypes as C

    import torch
    from paper_2005_09904_b200._capi import LUT_DP, LUT_NAIVE, KernelStats

    m, n, b, beta, mu = 300, 700, 3, 2, 10
    w = bq.random_uniform(m, n, 11)
    x = bq.random_normal(n, b, 12)
    layer = bq.PackedLinear.from_weights(w, beta, mu)
    keys, alpha = layer.export()
    kd = torch.from_numpy(keys.view(np.int16)).cuda()
    ad = torch.from_numpy(alpha).cuda()
    xd = torch.from_numpy(x).cuda()
    ws = torch.empty(int(bq.lib.bqg_biqgemm_exact_workspace_bytes(m, n, b, beta, mu)), dtype=torch.uint8,
                     device="cuda")
    ys = {}
    for builder in (LUT_DP, LUT_NAIVE):
        yd = torch.empty((m, b), device="cuda")
        st = KernelStats()
        bq.check(bq.lib.bqg_biqgemm_exact_ex_f32(kd.data_ptr(), ad.data_ptr(), xd.data_ptr(), n, yd.data_ptr(), m, n,
                                                b, beta, mu, builder, ws.data_ptr(), ws.numel(), C.byref(st), None))
        G = (n + mu - 1) // mu
        per = (1 << mu) * mu if builder == LUT_NAIVE else (1 << mu) + mu - 1
        assert st.lut_build_ops == per * G * b
        assert st.build_seconds > 0 and st.query_seconds > 0
        ys[builder] = yd.cpu().numpy()
    assert np.array_equal(ys[LUT_DP], layer.forward(x, exact=True))
    fast = KernelStats()
    layer2 = bq.PackedLinear.from_weights(w, beta, 8)
    layer2.forward(x, stats=fast)
    assert fast.build_seconds == 0 and fast.query_seconds > 0  # fused: the build runs inside the query kernel
    layer.close()
    layer2.close()
