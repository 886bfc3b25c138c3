// Scale-invariant SAI loss, forward and dL/dg (training.py:57-94; autodiff.py:190-239, 265-303).
//
// G side (t = G^T w, u = G t + eps w) in the reference's double roundings and orders.  The
// A side is evaluated by the reference in x87 long double (64-bit significand); here it runs in
// double-double (~106-bit), i.e. at least as accurate, with the same roundings to double at the
// same places (row sums of A u are rounded to double because the reference stores them in a
// float64 array, sparse.py:178; z is rounded to double for the backward pass, autodiff.py:291).
// Backward follows the tape closures in order: du = A^T(2 inv_norm z) (np.add.at order),
// v = G^T du, dg = du[row] t[col] + w[row] v[col].
#include "spmv.cuh"

namespace sg {

struct dd { double hi, lo; };

__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div_d(dd a, dd b) {  // a / b
  double q1 = a.hi / b.hi;
  dd r = dd_add(a, dd_mul(b, dd{-q1, 0.0}));
  double q2 = r.hi / b.hi;
  r = dd_add(r, dd_mul(b, dd{-q2, 0.0}));
  double q3 = r.hi / b.hi;
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}
__device__ __forceinline__ dd dd_sqrt(dd a) {
  if (a.hi <= 0.0) return {0.0, 0.0};
  double x = sqrt(a.hi);
  dd xx = two_prod(x, x);
  dd r = dd_add(a, dd{-xx.hi, -xx.lo});
  return quick_two_sum(x, r.hi / (2.0 * x));
}

// Deterministic block reduction of a dd value (fixed tree over shared memory).
__device__ dd block_dd_sum(dd v, dd* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = dd_add(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  dd r = sh[0];
  __syncthreads();
  return r;
}

constexpr int LT = 256;

// kind 0: |a| (sum; then / nnz), 1: a*a exact (sum; then sqrt), 2: |a| (sum)
__global__ void __launch_bounds__(LT) k_norm_dd_partial(const double* __restrict__ a, int64_t nnz,
                                                        int kind, dd* part) {
  __shared__ dd sh[LT];
  dd acc{0.0, 0.0};
  for (int64_t k = blockIdx.x * (int64_t)LT + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * LT) {
    const double v = a[k];
    acc = dd_add(acc, kind == 1 ? two_prod(v, v) : dd{fabs(v), 0.0});
  }
  dd r = block_dd_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

__global__ void __launch_bounds__(LT) k_norm_dd_finish(const dd* part, int nparts, int64_t nnz,
                                                       int kind, dd* norm) {
  __shared__ dd sh[LT];
  dd acc{0.0, 0.0};
  for (int k = threadIdx.x; k < nparts; k += LT) acc = dd_add(acc, part[k]);
  dd r = block_dd_sum(acc, sh);
  if (threadIdx.x == 0) {
    if (kind == 0) r = dd_div_d(r, dd{(double)nnz, 0.0});
    else if (kind == 1) r = dd_sqrt(r);
    *norm = r;
  }
}

// y_i = double(sum_k a_ik u_k) (dd accumulation); z_i = y_i / norm - w_i (dd); z64; sum z^2.
__global__ void __launch_bounds__(LT) k_loss_rows(int64_t n, const int32_t* __restrict__ offs,
                                                  const int32_t* __restrict__ cols,
                                                  const double* __restrict__ vals,
                                                  const double* __restrict__ u,
                                                  const double* __restrict__ w, const dd* norm_p,
                                                  double* z64, dd* part) {
  __shared__ dd sh[LT];
  const dd norm = *norm_p;
  dd acc{0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)LT + threadIdx.x; i < n; i += (int64_t)gridDim.x * LT) {
    dd y{0.0, 0.0};
    for (int32_t k = offs[i]; k < offs[i + 1]; ++k) y = dd_add(y, two_prod(vals[k], u[cols[k]]));
    const double y64 = y.hi + y.lo;  // rounded to double (normalised dd => hi + lo rounds to hi)
    dd z = dd_add(dd_div_d(dd{y64, 0.0}, norm), dd{-w[i], 0.0});
    z64[i] = z.hi + z.lo;
    acc = dd_add(acc, dd_mul(z, z));
  }
  dd r = block_dd_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

__global__ void __launch_bounds__(LT) k_loss_finish(const dd* part, int nparts, const dd* norm_p,
                                                    double* out) {
  __shared__ dd sh[LT];
  dd acc{0.0, 0.0};
  for (int k = threadIdx.x; k < nparts; k += LT) acc = dd_add(acc, part[k]);
  dd r = block_dd_sum(acc, sh);
  if (threadIdx.x == 0) {
    out[0] = r.hi + r.lo;
    const dd inv = dd_div_d(dd{1.0, 0.0}, *norm_p);
    out[1] = inv.hi + inv.lo;  // float(1 / norm_ld)
  }
}

__global__ void k_dz(int64_t n, const double* __restrict__ z64, const double* __restrict__ scal,
                     double* dz) {
  const double c = mul(2.0, scal[1]);  // (2.0 * 1.0 * inv_norm)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dz[i] = mul(c, z64[i]);
}

__global__ void k_grad(int64_t nnz, const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                       const double* __restrict__ du, const double* __restrict__ t,
                       const double* __restrict__ w, const double* __restrict__ v, double* grad) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[k], c = cols[k];
    grad[k] = add(mul(du[r], t[c]), mul(w[r], v[c]));
  }
}

constexpr int kRows = 256;
constexpr int kCap = 2048;

template <int ORDER>
__global__ void __launch_bounds__(kRows) k_loss_spmv(int64_t n, const int32_t* __restrict__ offs,
                                                     const int32_t* __restrict__ cols,
                                                     const double* __restrict__ vals,
                                                     const double* __restrict__ x,
                                                     const double* __restrict__ addv, double eps,
                                                     double* __restrict__ y) {
  __shared__ RowTile<kRows, kCap> t;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int64_t r1 = r0 + kRows < n ? r0 + kRows : n;
  stage_rows(t, r0, r1, offs, cols, vals);
  const int lr = threadIdx.x;
  if (r0 + lr < r1) {
    double v = tile_row_dot<ORDER, false, 0>(t, lr, cols, vals, XF{x, nullptr, 0.0});
    if (addv) v = add(v, mul(eps, addv[r0 + lr]));
    y[r0 + lr] = v;
  }
}

}  // namespace sg

using namespace sg;

extern "C" int sg_sai_loss(int64_t n, const int32_t* a_offs, const int32_t* a_cols,
                           const double* a_vals, const int32_t* at_offs, const int32_t* at_cols,
                           const double* at_vals, const int32_t* g_offs, const int32_t* g_cols,
                           const double* g_vals, const int32_t* gt_offs, const int32_t* gt_cols,
                           const double* gt_vals, const int32_t* g_rows, double eps,
                           const double* w, int norm_kind, double* loss_host, double* grad_out,
                           void* ws, size_t* ws_bytes, void* stream) {
  const int NP = 148 * 4;
  Carve c(ws);
  double* t = c.take<double>(n + 2);
  double* u = c.take<double>(n + 2);
  double* z64 = c.take<double>(n + 2);
  double* du = c.take<double>(n + 2);
  double* v = c.take<double>(n + 2);
  dd* part = c.take<dd>(NP);
  dd* norm = c.take<dd>(1);
  double* scal = c.take<double>(2);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  if (norm_kind < 0 || norm_kind > 2) { set_error("unknown norm kind"); return SG_EINVAL; }
  if (n <= 0) { set_error("empty system"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  int64_t a_nnz = 0, g_nnz = 0;
  {
    int32_t h[2];
    SG_CUDA(cudaMemcpyAsync(&h[0], a_offs + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaMemcpyAsync(&h[1], g_offs + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    a_nnz = h[0];
    g_nnz = h[1];
  }
  if (a_nnz == 0) { set_error("matrix norm is zero"); return SG_EINVAL; }
  const unsigned gr = (unsigned)ceil_div(n, kRows);
  k_loss_spmv<kOrderSeq><<<gr, kRows, 0, s>>>(n, gt_offs, gt_cols, gt_vals, w, nullptr, 0.0, t);
  k_loss_spmv<kOrderNumpy><<<gr, kRows, 0, s>>>(n, g_offs, g_cols, g_vals, t, w, eps, u);
  k_norm_dd_partial<<<NP, LT, 0, s>>>(a_vals, a_nnz, norm_kind, part);
  k_norm_dd_finish<<<1, LT, 0, s>>>(part, NP, a_nnz, norm_kind, norm);
  k_loss_rows<<<NP, LT, 0, s>>>(n, a_offs, a_cols, a_vals, u, w, norm, z64, part);
  k_loss_finish<<<1, LT, 0, s>>>(part, NP, norm, scal);
  SG_LAUNCH_CHECK("sai loss forward");
  if (grad_out) {
    k_dz<<<NP, LT, 0, s>>>(n, z64, scal, z64);
    k_loss_spmv<kOrderSeq><<<gr, kRows, 0, s>>>(n, at_offs, at_cols, at_vals, z64, nullptr, 0.0, du);
    k_loss_spmv<kOrderSeq><<<gr, kRows, 0, s>>>(n, gt_offs, gt_cols, gt_vals, du, nullptr, 0.0, v);
    if (g_nnz > 0) k_grad<<<NP, LT, 0, s>>>(g_nnz, g_rows, g_cols, du, t, w, v, grad_out);
    SG_LAUNCH_CHECK("sai loss backward");
  }
  double h[2];
  dd nh;
  SG_CUDA(cudaMemcpyAsync(h, scal, sizeof(h), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaMemcpyAsync(&nh, norm, sizeof(dd), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  if (nh.hi == 0.0) { set_error("matrix norm is zero"); return SG_EINVAL; }  // autodiff.py:285
  *loss_host = h[0];
  return SG_OK;
}

// ------------------------------------------------------------------ row-partitioned loss
// The SAI loss of ONE system split like the row-partitioned PCG (BASELINE
// configs[4] asks for the loss forward and backward on the partition).  Each partition works on
// its extended local system (owned rows + 3 half-bandwidths of ghost rows): t, u and z come out
// exact on the owned rows; the caller copies the neighbours' owned z into the ghost rows (the one
// halo of the loss), after which du, v and dL/dg are exact for every entry of the owned rows.
// The norm and the loss are dd sums over owned entries / rows, combined in partition order.
namespace sg {

__global__ void __launch_bounds__(LT) k_loss_rows_own(int64_t n, int64_t own_lo, int64_t own_hi,
                                                      const int32_t* __restrict__ offs,
                                                      const int32_t* __restrict__ cols,
                                                      const double* __restrict__ vals, const double* __restrict__ u,
                                                      const double* __restrict__ w, const dd* norm_p, double* z64,
                                                      dd* part) {
  __shared__ dd sh[LT];
  const dd norm = *norm_p;
  dd acc{0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)LT + threadIdx.x; i < n; i += (int64_t)gridDim.x * LT) {
    dd y{0.0, 0.0};
    for (int32_t k = offs[i]; k < offs[i + 1]; ++k) y = dd_add(y, two_prod(vals[k], u[cols[k]]));
    const double y64 = y.hi + y.lo;
    dd z = dd_add(dd_div_d(dd{y64, 0.0}, norm), dd{-w[i], 0.0});
    z64[i] = z.hi + z.lo;
    if (i >= own_lo && i < own_hi) acc = dd_add(acc, dd_mul(z, z));
  }
  dd r = block_dd_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = r;
}

__global__ void __launch_bounds__(LT) k_dd_reduce(const dd* part, int nparts, dd* out) {
  __shared__ dd sh[LT];
  dd acc{0.0, 0.0};
  for (int k = threadIdx.x; k < nparts; k += LT) acc = dd_add(acc, part[k]);
  dd r = block_dd_sum(acc, sh);
  if (threadIdx.x == 0) *out = r;
}

// partition partials (dd) in partition order; kind transform; out = {norm hi, norm lo, 1/norm}
__global__ void k_norm_combine(const dd* parts, int P, int64_t nnz, int kind, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  dd r{0.0, 0.0};
  for (int p = 0; p < P; ++p) r = dd_add(r, parts[p]);
  if (kind == 0) r = dd_div_d(r, dd{(double)nnz, 0.0});
  else if (kind == 1) r = dd_sqrt(r);
  out[0] = r.hi;
  out[1] = r.lo;
  const dd inv = dd_div_d(dd{1.0, 0.0}, r);
  out[2] = inv.hi + inv.lo;
}

__global__ void k_dd_sum_parts(const dd* parts, int P, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  dd r{0.0, 0.0};
  for (int p = 0; p < P; ++p) r = dd_add(r, parts[p]);
  *out = r.hi + r.lo;
}

}  // namespace sg

extern "C" int sg_loss_norm_partial(const double* vals, int64_t nnz, int kind, double* part_out, void* ws,
                                    size_t* ws_bytes, void* stream) {
  const int NP = 148 * 4;
  Carve c(ws);
  dd* part = c.take<dd>(NP);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (kind < 0 || kind > 2) { set_error("unknown norm kind"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  k_norm_dd_partial<<<NP, LT, 0, s>>>(vals, nnz > 0 ? nnz : 0, kind, part);
  k_dd_reduce<<<1, LT, 0, s>>>(part, NP, reinterpret_cast<dd*>(part_out));
  SG_LAUNCH_CHECK("loss norm partial");
  return SG_OK;
}

extern "C" int sg_loss_norm_combine(const double* parts, int32_t n_parts, int64_t nnz_total, int kind,
                                    double* norm3_out, void* stream) {
  if (n_parts < 1 || nnz_total < 1) { set_error("matrix norm is zero"); return SG_EINVAL; }
  k_norm_combine<<<1, 32, 0, as_stream(stream)>>>(reinterpret_cast<const dd*>(parts), n_parts, nnz_total, kind,
                                                  norm3_out);
  SG_LAUNCH_CHECK("loss norm combine");
  return SG_OK;
}

extern "C" int sg_sai_loss_part_fwd(int64_t n, const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                                    const int32_t* g_offs, const int32_t* g_cols, const double* g_vals,
                                    const int32_t* gt_offs, const int32_t* gt_cols, const double* gt_vals,
                                    double eps, const double* w, const double* norm3, int64_t own_lo,
                                    int64_t own_hi, double* t_out, double* z64_out, double* part_out, void* ws,
                                    size_t* ws_bytes, void* stream) {
  const int NP = 148 * 4;
  Carve c(ws);
  double* u = c.take<double>(n + 2);
  dd* part = c.take<dd>(NP);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  if (n <= 0 || !(0 <= own_lo && own_lo < own_hi && own_hi <= n)) { set_error("bad owned row range"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  const unsigned gr = (unsigned)ceil_div(n, kRows);
  k_loss_spmv<kOrderSeq><<<gr, kRows, 0, s>>>(n, gt_offs, gt_cols, gt_vals, w, nullptr, 0.0, t_out);
  k_loss_spmv<kOrderNumpy><<<gr, kRows, 0, s>>>(n, g_offs, g_cols, g_vals, t_out, w, eps, u);
  k_loss_rows_own<<<NP, LT, 0, s>>>(n, own_lo, own_hi, a_offs, a_cols, a_vals, u, w,
                                    reinterpret_cast<const dd*>(norm3), z64_out, part);
  k_dd_reduce<<<1, LT, 0, s>>>(part, NP, reinterpret_cast<dd*>(part_out));
  SG_LAUNCH_CHECK("partitioned sai loss forward");
  return SG_OK;
}

extern "C" int sg_loss_sum_parts(const double* parts, int32_t n_parts, double* loss_host, void* stream) {
  cudaStream_t s = as_stream(stream);
  double* out = nullptr;
  SG_CUDA(cudaMallocAsync(&out, sizeof(double), s));
  k_dd_sum_parts<<<1, 32, 0, s>>>(reinterpret_cast<const dd*>(parts), n_parts, out);
  SG_LAUNCH_CHECK("loss sum");
  SG_CUDA(cudaMemcpyAsync(loss_host, out, sizeof(double), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaFreeAsync(out, s));
  SG_CUDA(cudaStreamSynchronize(s));
  return SG_OK;
}

extern "C" int sg_sai_loss_part_bwd(int64_t n, const int32_t* at_offs, const int32_t* at_cols, const double* at_vals,
                                    const int32_t* gt_offs, const int32_t* gt_cols, const double* gt_vals,
                                    const int32_t* g_offs, const int32_t* g_rows, const int32_t* g_cols,
                                    const double* w, const double* t, const double* z64, const double* norm3,
                                    int64_t own_lo, int64_t own_hi, double* grad_out, void* ws, size_t* ws_bytes,
                                    void* stream) {
  const int NP = 148 * 4;
  Carve c(ws);
  double* dz = c.take<double>(n + 2);
  double* du = c.take<double>(n + 2);
  double* v = c.take<double>(n + 2);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  if (n <= 0 || !(0 <= own_lo && own_lo < own_hi && own_hi <= n)) { set_error("bad owned row range"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  int32_t e[2];
  SG_CUDA(cudaMemcpyAsync(&e[0], g_offs + own_lo, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaMemcpyAsync(&e[1], g_offs + own_hi, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  const unsigned gr = (unsigned)ceil_div(n, kRows);
  k_dz<<<NP, LT, 0, s>>>(n, z64, norm3 + 1, dz);  // scal[1] = norm3[2] = 1 / norm
  k_loss_spmv<kOrderSeq><<<gr, kRows, 0, s>>>(n, at_offs, at_cols, at_vals, dz, nullptr, 0.0, du);
  k_loss_spmv<kOrderSeq><<<gr, kRows, 0, s>>>(n, gt_offs, gt_cols, gt_vals, du, nullptr, 0.0, v);
  if (e[1] > e[0])
    k_grad<<<NP, LT, 0, s>>>(e[1] - e[0], g_rows + e[0], g_cols + e[0], du, t, w, v, grad_out + e[0]);
  SG_LAUNCH_CHECK("partitioned sai loss backward");
  return SG_OK;
}
