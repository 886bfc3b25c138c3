// Standalone SpMV entry points (sparse.py:186-201, precond.py:143-145).
#include "spmv.cuh"

namespace sg {

constexpr int kRows = 256;
constexpr int kCap = 2048;

template <int ORDER>
__global__ void __launch_bounds__(kRows) k_spmv(int64_t n, const int32_t* __restrict__ offs,
                                                const int32_t* __restrict__ cols,
                                                const double* __restrict__ vals,
                                                const double* __restrict__ x, double* __restrict__ y) {
  __shared__ RowTile<kRows, kCap> t;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int64_t r1 = r0 + kRows < n ? r0 + kRows : n;
  stage_rows(t, r0, r1, offs, cols, vals);
  const int lr = threadIdx.x;
  if (r0 + lr < r1)
    y[r0 + lr] = tile_row_dot<ORDER, false, 0>(t, lr, cols, vals, XF{x, nullptr, 0.0});
}

// Long rows (>= 32 entries on average): one warp per row in numpy's exact order (warp_row_numpy).
constexpr int kWarpCta = 8;
__global__ void __launch_bounds__(32 * kWarpCta) k_spmv_warp(int64_t n, const int32_t* __restrict__ offs,
                                                             const int32_t* __restrict__ cols,
                                                             const double* __restrict__ vals,
                                                             const double* __restrict__ x, double* __restrict__ y) {
  __shared__ int2 leaf[kWarpCta][kWarpLeaves];
  __shared__ double lsum[kWarpCta][kWarpLeaves];
  const int w = threadIdx.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * kWarpCta + w; i < n; i += (int64_t)gridDim.x * kWarpCta) {
    const double v = warp_row_numpy<0>(vals, cols, offs[i], offs[i + 1], XF{x, nullptr, 0.0}, leaf[w], lsum[w]);
    if ((threadIdx.x & 31) == 0) y[i] = v;
  }
}

// s = spmv(G, t) + eps * r
__global__ void __launch_bounds__(kRows) k_apply_g(int64_t n, const int32_t* __restrict__ offs,
                                                   const int32_t* __restrict__ cols,
                                                   const double* __restrict__ vals,
                                                   const double* __restrict__ tv, double eps,
                                                   const double* __restrict__ r, double* __restrict__ s) {
  __shared__ RowTile<kRows, kCap> t;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int64_t r1 = r0 + kRows < n ? r0 + kRows : n;
  stage_rows(t, r0, r1, offs, cols, vals);
  const int lr = threadIdx.x;
  if (r0 + lr < r1) {
    const double y = tile_row_dot<kOrderNumpy, false, 0>(t, lr, cols, vals, XF{tv, nullptr, 0.0});
    s[r0 + lr] = add(y, mul(eps, r[r0 + lr]));
  }
}

// out = a + c*b (mode 0) or a - c*b (mode 1), each product rounded first (numpy semantics).
__global__ void k_axpby(double* __restrict__ out, const double* __restrict__ a, const double* __restrict__ b,
                        double c, int64_t n, int mode) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double p = mul(c, b[i]);
    out[i] = mode == 0 ? add(a[i], p) : sub(a[i], p);
  }
}

// Deterministic dot product: fixed grid, fixed per-thread strides, fixed trees.
constexpr int kDotBlocks = 296;
__global__ void k_dot_partial(const double* __restrict__ x, const double* __restrict__ y, int64_t n, double* part) {
  __shared__ double red[8];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = add(s, mul(x[i], y[i]));
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_dot_final(const double* __restrict__ part, int np, double* out) {
  __shared__ double red[8];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s = add(s, part[i]);
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

}  // namespace sg

using namespace sg;

extern "C" int sg_axpby(double* out, const double* a, const double* b, double c, int64_t n, int mode, void* stream) {
  if (n <= 0) return SG_OK;
  const int64_t g = ceil_div(n, 256);
  k_axpby<<<(unsigned)(g < 148 * 16 ? g : 148 * 16), 256, 0, as_stream(stream)>>>(out, a, b, c, n, mode);
  SG_LAUNCH_CHECK("k_axpby");
  return SG_OK;
}

extern "C" int sg_dot(const double* x, const double* y, int64_t n, double* out, void* ws, size_t* ws_bytes,
                      void* stream) {
  Carve c(ws);
  double* part = c.take<double>(kDotBlocks);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  cudaStream_t s = as_stream(stream);
  k_dot_partial<<<kDotBlocks, 256, 0, s>>>(x, y, n, part);
  k_dot_final<<<1, 256, 0, s>>>(part, kDotBlocks, out);
  SG_LAUNCH_CHECK("k_dot");
  return SG_OK;
}

extern "C" int sg_spmv(int64_t n_rows, const int32_t* offs, const int32_t* cols, const double* vals,
                       const double* x, double* y, void* stream) {
  if (n_rows <= 0) return SG_OK;
  k_spmv<kOrderNumpy><<<(unsigned)ceil_div(n_rows, kRows), kRows, 0, as_stream(stream)>>>(
      n_rows, offs, cols, vals, x, y);
  SG_LAUNCH_CHECK("k_spmv<numpy>");
  return SG_OK;
}

extern "C" int sg_spmv_warp(int64_t n_rows, const int32_t* offs, const int32_t* cols, const double* vals,
                            const double* x, double* y, void* stream) {
  if (n_rows <= 0) return SG_OK;
  const int64_t g = ceil_div(n_rows, kWarpCta);
  k_spmv_warp<<<(unsigned)(g < 148 * 64 ? g : 148 * 64), 32 * kWarpCta, 0, as_stream(stream)>>>(n_rows, offs, cols,
                                                                                             vals, x, y);
  SG_LAUNCH_CHECK("k_spmv_warp");
  return SG_OK;
}

extern "C" int sg_spmv_seq(int64_t n_rows, const int32_t* offs, const int32_t* cols,
                           const double* vals, const double* x, double* y, void* stream) {
  if (n_rows <= 0) return SG_OK;
  k_spmv<kOrderSeq><<<(unsigned)ceil_div(n_rows, kRows), kRows, 0, as_stream(stream)>>>(
      n_rows, offs, cols, vals, x, y);
  SG_LAUNCH_CHECK("k_spmv<seq>");
  return SG_OK;
}

extern "C" int sg_learned_apply(int64_t n, const int32_t* g_offs, const int32_t* g_cols,
                                const double* g_vals, const int32_t* gt_offs,
                                const int32_t* gt_cols, const double* gt_vals, double eps,
                                const double* r, double* t_ws, double* s_out, void* stream) {
  if (n <= 0) return SG_OK;
  cudaStream_t s = as_stream(stream);
  const unsigned g = (unsigned)ceil_div(n, kRows);
  k_spmv<kOrderSeq><<<g, kRows, 0, s>>>(n, gt_offs, gt_cols, gt_vals, r, t_ws);
  SG_LAUNCH_CHECK("k_spmv<seq>");
  k_apply_g<<<g, kRows, 0, s>>>(n, g_offs, g_cols, g_vals, t_ws, eps, r, s_out);
  SG_LAUNCH_CHECK("k_apply_g");
  return SG_OK;
}
