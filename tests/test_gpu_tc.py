"""GPU: the tcgen05 building block of the tensor-core GNN path -- one 128-row tile on the 5th-
generation tensor core (kind::tf32, shared-memory operand descriptors, TMEM accumulator) -- against
an fp64 host product.  3xTF32 must reach fp32 accuracy (the north_star's fp32 bar for G is 1e-5)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2510_27517_b200 import _lib as L  # noqa: E402


def _tile(a, w, split3):
    k, n = w.shape
    ad = torch.as_tensor(a, dtype=torch.float32, device="cuda").contiguous()
    wd = torch.as_tensor(w, dtype=torch.float32, device="cuda").contiguous()
    out = torch.zeros(128 * n, dtype=torch.float32, device="cuda")
    L.check(L.lib().sg_tc_gemm_selftest(L.ptr(ad), L.ptr(wd), k, n, split3, L.ptr(out), L.stream_ptr()))
    return out.cpu().numpy().reshape(128, n)


@pytest.mark.parametrize("k,n", [(24, 24), (8, 8), (32, 32), (24, 1), (17, 13)])
def test_tcgen05_tf32_tile(k, n):
    rng = np.random.default_rng(k * 100 + n)
    a = rng.standard_normal((128, k)).astype(np.float32)
    w = rng.standard_normal((k, n)).astype(np.float32)
    ref = a.astype(np.float64) @ w.astype(np.float64)
    scale = np.abs(a).astype(np.float64) @ np.abs(w).astype(np.float64)
    err3 = np.max(np.abs(_tile(a, w, 1) - ref) / scale)
    err1 = np.max(np.abs(_tile(a, w, 0) - ref) / scale)
    assert err3 < 2e-6, err3       # 3xTF32 ~ fp32
    assert err1 < 2e-3, err1       # plain TF32 (10-bit mantissa)
    assert err1 > err3
