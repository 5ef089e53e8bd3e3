"""GPU comparison baselines (reference baselines.hpp): gemm_unpack equals
the BiQGEMM result within the fp32 contract (the reference's own
test_baselines.cpp:70-76 pins unpack == LUT), and the bandwidth probe
computes the reference's (meaningless) per-row word products."""
import numpy as np
import pytest

from test_gpu_parity import assert_close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,b,beta", [(1, 1, 1, 1), (33, 70, 1, 2), (200, 777, 3, 3), (4096, 4096, 1, 3),
                                        (100, 300, 8, 2)])
def test_gemm_unpack_matches_reference_math(bq, port, cuda, m, n, b, beta):
    import torch

    w = bq.random_uniform(m, n, 7 + m)
    x = bq.random_normal(n, b, 8 + n)
    layer = bq.PackedLinear.from_weights(w, beta, 8)
    keys, alpha, planes = layer.export(planes=True)
    y_ref, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, 8, x)
    y = torch.empty((m, b), device="cuda")
    bq.gemm_unpack_device(torch.from_numpy(planes.view(np.int32)).cuda(), torch.from_numpy(alpha).cuda(),
                          torch.from_numpy(x).cuda(), y, m, n, beta)
    torch.cuda.synchronize()
    assert_close(y.cpu().numpy(), y_ref)
    # plane mode (alpha = 1)
    y1 = torch.empty((m, b), device="cuda")
    bq.gemm_unpack_device(torch.from_numpy(planes[:1].view(np.int32)).cuda(), None, torch.from_numpy(x).cuda(), y1,
                          m, n, 1)
    torch.cuda.synchronize()
    y1_ref, _ = port.biqgemm(keys[:1].astype(np.uint32), None, n, 8, x)
    assert_close(y1.cpu().numpy(), y1_ref)
    layer.close()


def test_bandwidth_probe_arithmetic(bq, cuda):
    import torch

    m, n = 64, 300
    wpr = (n + 31) // 32
    rng = np.random.default_rng(3)
    words = rng.integers(0, 2**32, size=(m, wpr), dtype=np.uint64).astype(np.uint32)
    x = bq.random_normal(n, 1, 4)
    out = torch.empty(m, device="cuda")
    bq.bandwidth_probe_device(torch.from_numpy(words.view(np.int32)).cuda(), m, n, torch.from_numpy(x).cuda(), out,
                              streaming=False)
    torch.cuda.synchronize()
    xs = x[:, 0].astype(np.float64)
    ref = (words.astype(np.float64) * xs[(np.arange(wpr) * 32) % n][None, :]).sum(1).astype(np.float32)
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-6)
    out2 = torch.empty(1184 * 512, device="cuda")
    bq.bandwidth_probe_device(torch.from_numpy(words.view(np.int32)).cuda(), m, n, torch.from_numpy(x).cuda(), out2)
    torch.cuda.synchronize()
