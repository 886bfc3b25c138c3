// Device primitives of the GNN training step (GNN backward + AdamW,
// replacing the reference's tape closures autodiff.py:63-177 and training.py:126-147).
//
// The training forward keeps every intermediate the backward needs (pre-activations, node
// states per layer, edge states per layer) and the backward is a fixed sequence of these
// primitives (composed in training.py).  The graphs the reference trains on are small
// (heat2d 16x16: 256 nodes, 1216 edges), so these are plain fp64 kernels written for
// determinism, not tensor-core throughput:
//   * every row-wise product / reduction runs in a fixed order;
//   * parameter gradients (sums over nodes or edges of outer products) are reduced in two
//     fixed-shape passes (per-block partials, then one ordered sum), so a training run is
//     bit-reproducible run to run (the reference's determinism test, test_training.py:250-260).
#include "common.cuh"

namespace sg {

// out[r][c] = act( sum_k in[r][k] * W[k][c] (+ b[c]) ) (+ add[r][c]); in row stride ldi, W row
// stride ldw (so a row block of a larger matrix can be used), out row stride ldo.
// TRANS: W is applied transposed (out[r][c] = sum_k in[r][k] * W[c][k]).
template <bool TRANS>
__global__ void k_affine(int64_t N, int din, int dout, const double* __restrict__ in, int ldi,
                         const double* __restrict__ W, int ldw, const double* __restrict__ b,
                         const double* add, double* out, int ldo, int relu) {  // add may alias out
  const int64_t total = N * dout;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / dout;
    const int c = (int)(idx % dout);
    double s = 0.0;
    for (int k = 0; k < din; ++k) s = fma(in[r * ldi + k], TRANS ? W[(int64_t)c * ldw + k] : W[(int64_t)k * ldw + c], s);
    if (b) s += b[c];
    if (relu) s = s > 0.0 ? s : 0.0;
    if (add) s += add[r * ldo + c];
    out[r * ldo + c] = s;
  }
}

// pre[e][c] = P[row_e][c] + Q[col_e][c] + (e_feat[e] * crow[c]) + (H[e][c]) + b[c]
__global__ void k_edge_pre(int64_t E, int d, const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                           const double* __restrict__ P, const double* __restrict__ Q,
                           const double* __restrict__ ef, const double* __restrict__ crow,
                           const double* __restrict__ H, const double* __restrict__ b, double* __restrict__ pre) {
  const int64_t total = E * d;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = idx / d;
    const int c = (int)(idx % d);
    double s = P[(int64_t)rows[e] * d + c] + Q[(int64_t)cols[e] * d + c];
    if (crow) s += ef[e] * crow[c];
    if (H) s += H[idx];
    if (b) s += b[c];
    pre[idx] = s;
  }
}

// dst = src * [pre > 0] (elementwise; dst may alias src)
__global__ void k_relu_grad(int64_t M, const double* __restrict__ pre, const double* src, double* dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = pre[i] > 0.0 ? src[i] : 0.0;
}

// dst[i][c] (+)= sum over the entries of segment i (CSR offs; perm maps segment positions to
// source rows, or identity when null) of src[k][c], in segment order.
__global__ void k_segment_sum(int64_t n, int d, const int32_t* __restrict__ offs, const int32_t* __restrict__ perm,
                              const double* __restrict__ src, double* __restrict__ dst, int accumulate) {
  const int64_t total = n * d;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / d;
    const int c = (int)(idx % d);
    double s = accumulate ? dst[idx] : 0.0;
    for (int32_t k = offs[i]; k < offs[i + 1]; ++k) s += src[(int64_t)(perm ? perm[k] : k) * d + c];
    dst[idx] = s;
  }
}

// Deterministic sum over rows of outer products: part[blk][a][b] = sum_{r in chunk blk}
// A[r][a] * B[r][b] (A == null -> ones column, i.e. column sums of B; wA = 1).
constexpr int kOuterRows = 1024;  // rows per partial
__global__ void k_outer_partial(int64_t N, int da, int db, const double* __restrict__ A, int lda,
                                const double* __restrict__ B, int ldb, double* __restrict__ part) {
  const int64_t r0 = (int64_t)blockIdx.x * kOuterRows;
  const int64_t r1 = r0 + kOuterRows < N ? r0 + kOuterRows : N;
  for (int idx = threadIdx.x; idx < da * db; idx += blockDim.x) {
    const int a = idx / db, bcol = idx % db;
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) s = fma(A ? A[r * lda + a] : 1.0, B[r * ldb + bcol], s);
    part[(int64_t)blockIdx.x * da * db + idx] = s;
  }
}

__global__ void k_outer_reduce(int nblk, int m, const double* __restrict__ part, double* __restrict__ out,
                               int accumulate) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < m; idx += gridDim.x * blockDim.x) {
    double s = accumulate ? out[idx] : 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * m + idx];
    out[idx] = s;
  }
}

// AdamW (training.py:126-147) with numpy's roundings (no contraction): m, v, params in place.
// g is divided by gdiv first (the reference's grad_sum / len(batch)).
__global__ void k_adamw(int64_t n, double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                        double* __restrict__ v, double lr, double wd, double b1, double b2, double eps, double c1,
                        double c2, double gdiv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = __ddiv_rn(g[i], gdiv);
    const double mi = add(mul(b1, m[i]), mul(1.0 - b1, gi));
    const double vi = add(mul(b2, v[i]), mul(mul(1.0 - b2, gi), gi));
    m[i] = mi;
    v[i] = vi;
    const double mh = __ddiv_rn(mi, c1), vh = __ddiv_rn(vi, c2);
    const double upd = add(__ddiv_rn(mh, add(__dsqrt_rn(vh), eps)), mul(wd, p[i]));
    p[i] = sub(p[i], mul(lr, upd));
  }
}

static int grid_of(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace sg

using namespace sg;

extern "C" int sg_dense_affine(int64_t N, int32_t din, int32_t dout, const double* in, int32_t ldi, const double* W,
                               int32_t ldw, int32_t transpose_w, const double* b, const double* add, double* out,
                               int32_t ldo, int32_t relu, void* stream) {
  if (N < 0 || din < 0 || dout < 1) { set_error("bad affine shape"); return SG_EINVAL; }
  if (N == 0) return SG_OK;
  cudaStream_t s = as_stream(stream);
  if (transpose_w)
    k_affine<true><<<grid_of(N * dout), 256, 0, s>>>(N, din, dout, in, ldi, W, ldw, b, add, out, ldo, relu);
  else
    k_affine<false><<<grid_of(N * dout), 256, 0, s>>>(N, din, dout, in, ldi, W, ldw, b, add, out, ldo, relu);
  SG_LAUNCH_CHECK("k_affine");
  return SG_OK;
}

extern "C" int sg_edge_pre(int64_t E, int32_t d, const int32_t* rows, const int32_t* cols, const double* P,
                           const double* Q, const double* ef, const double* crow, const double* H, const double* b,
                           double* pre, void* stream) {
  if (E == 0) return SG_OK;
  k_edge_pre<<<grid_of(E * d), 256, 0, as_stream(stream)>>>(E, d, rows, cols, P, Q, ef, crow, H, b, pre);
  SG_LAUNCH_CHECK("k_edge_pre");
  return SG_OK;
}

extern "C" int sg_relu_grad(int64_t M, const double* pre, const double* src, double* dst, void* stream) {
  if (M == 0) return SG_OK;
  k_relu_grad<<<grid_of(M), 256, 0, as_stream(stream)>>>(M, pre, src, dst);
  SG_LAUNCH_CHECK("k_relu_grad");
  return SG_OK;
}

extern "C" int sg_segment_sum(int64_t n, int32_t d, const int32_t* offs, const int32_t* perm, const double* src,
                              double* dst, int32_t accumulate, void* stream) {
  if (n == 0) return SG_OK;
  k_segment_sum<<<grid_of(n * d), 256, 0, as_stream(stream)>>>(n, d, offs, perm, src, dst, accumulate);
  SG_LAUNCH_CHECK("k_segment_sum");
  return SG_OK;
}

extern "C" int sg_outer_sum(int64_t N, int32_t da, int32_t db, const double* A, int32_t lda, const double* B,
                            int32_t ldb, double* out, int32_t accumulate, void* ws, size_t* ws_bytes, void* stream) {
  const int64_t nblk = N > 0 ? (N + kOuterRows - 1) / kOuterRows : 1;
  const size_t need = (size_t)nblk * da * db * sizeof(double) + 256;
  if (ws == nullptr) { *ws_bytes = need; return SG_OK; }
  if (*ws_bytes < need) { set_error("outer_sum workspace too small"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  double* part = static_cast<double*>(ws);
  if (N == 0) {
    SG_CUDA(cudaMemsetAsync(part, 0, (size_t)da * db * sizeof(double), s));
  } else {
    k_outer_partial<<<(unsigned)nblk, 256, 0, s>>>(N, da, db, A, lda, B, ldb, part);
  }
  k_outer_reduce<<<grid_of(da * db), 256, 0, s>>>((int)nblk, da * db, part, out, accumulate);
  SG_LAUNCH_CHECK("k_outer_sum");
  return SG_OK;
}

extern "C" int sg_adamw(int64_t n, double* params, const double* grads, double* m, double* v, double lr, double wd,
                        double beta1, double beta2, double eps, int64_t t, double grad_div, void* stream) {
  if (t < 1) { set_error("step index is 1-based"); return SG_EINVAL; }
  const double c1 = 1.0 - pow(beta1, (double)t), c2 = 1.0 - pow(beta2, (double)t);
  k_adamw<<<grid_of(n), 256, 0, as_stream(stream)>>>(n, params, grads, m, v, lr, wd, beta1, beta2, eps, c1, c2,
                                                      grad_div);
  SG_LAUNCH_CHECK("k_adamw");
  return SG_OK;
}

// ------------------------------------------------------------------ FSAI construction
// build_fsai (precond.py:262-305) on the device, one thread per row: the
// local SPD system A[P_i, P_i] g = e_last over the row's lower pattern P_i (gathered from A's
// CSR by binary search), Cholesky (dense.py:56-69: pivots, then column updates), forward and
// back substitution (dense.py:72-93), g / sqrt(g_last); a non-positive / non-finite pivot falls
// back to 1/sqrt(a_ii) on the diagonal.  Patterns wider than kFsaiMax entries per row are
// reported (SG_EUNSUPPORTED) instead of solved.
namespace sg {
constexpr int kFsaiMax = 16;

__device__ double fsai_a(const int32_t* ao, const int32_t* ac, const double* av, int row, int col) {
  int lo = ao[row], hi = ao[row + 1];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (ac[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  return (lo < ao[row + 1] && ac[lo] == col) ? av[lo] : 0.0;
}

__global__ void k_fsai(int64_t n, const int32_t* __restrict__ ao, const int32_t* __restrict__ ac,
                       const double* __restrict__ av, const int32_t* __restrict__ lo_, const int32_t* __restrict__ lc,
                       double* __restrict__ lv, unsigned int* fallbacks, unsigned int* too_wide) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int p0 = lo_[i], m = lo_[i + 1] - p0;
    if (m > kFsaiMax) { atomicAdd(too_wide, 1u); continue; }
    double Lm[kFsaiMax][kFsaiMax];
    double y[kFsaiMax];
    bool ok = true;
    // Cholesky, column by column (dense.py:62-68)
    for (int j = 0; j < m && ok; ++j) {
      const int cj = lc[p0 + j];
      double dot = 0.0;
      for (int k = 0; k < j; ++k) dot = __dadd_rn(dot, __dmul_rn(Lm[j][k], Lm[j][k]));
      const double pivot = __dsub_rn(fsai_a(ao, ac, av, cj, cj), dot);
      if (!(pivot > 0.0) || !isfinite(pivot)) { ok = false; break; }
      Lm[j][j] = __dsqrt_rn(pivot);
      for (int r = j + 1; r < m; ++r) {
        double d2 = 0.0;
        for (int k = 0; k < j; ++k) d2 = __dadd_rn(d2, __dmul_rn(Lm[r][k], Lm[j][k]));
        Lm[r][j] = __ddiv_rn(__dsub_rn(fsai_a(ao, ac, av, lc[p0 + r], cj), d2), Lm[j][j]);
      }
    }
    if (ok) {
      // L y = e_last, then L^T g = y (g in place of y)
      for (int r = 0; r < m; ++r) {
        double s = 0.0;
        for (int k = 0; k < r; ++k) s = __dadd_rn(s, __dmul_rn(Lm[r][k], y[k]));
        y[r] = __ddiv_rn(__dsub_rn(r == m - 1 ? 1.0 : 0.0, s), Lm[r][r]);
      }
      for (int r = m - 1; r >= 0; --r) {
        double s = 0.0;
        for (int k = r + 1; k < m; ++k) s = __dadd_rn(s, __dmul_rn(Lm[k][r], y[k]));
        y[r] = __ddiv_rn(__dsub_rn(y[r], s), Lm[r][r]);
      }
      const double pv = y[m - 1];
      if (!(pv > 0.0) || !isfinite(pv)) ok = false;
      else {
        const double sc = __dsqrt_rn(pv);
        for (int r = 0; r < m; ++r) lv[p0 + r] = __ddiv_rn(y[r], sc);
      }
    }
    if (!ok) {
      atomicAdd(fallbacks, 1u);
      for (int r = 0; r < m - 1; ++r) lv[p0 + r] = 0.0;
      lv[p0 + m - 1] = __ddiv_rn(1.0, __dsqrt_rn(fsai_a(ao, ac, av, (int)i, (int)i)));
    }
  }
}
}  // namespace sg

extern "C" int sg_fsai_build(int64_t n, const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                             const int32_t* l_offs, const int32_t* l_cols, double* l_vals, int64_t* fallbacks_host,
                             void* stream) {
  cudaStream_t s = as_stream(stream);
  unsigned int* cnt = nullptr;
  SG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cnt), 2 * sizeof(unsigned int), s));
  SG_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned int), s));
  if (n > 0) {
    k_fsai<<<grid_of(n), 128, 0, s>>>(n, a_offs, a_cols, a_vals, l_offs, l_cols, l_vals, cnt, cnt + 1);
    SG_LAUNCH_CHECK("k_fsai");
  }
  unsigned int h[2] = {0, 0};
  SG_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(cnt, s);
  if (h[1]) {
    set_error("FSAI: %u rows have more than %d lower-pattern entries", h[1], kFsaiMax);
    return SG_EUNSUPPORTED;
  }
  if (fallbacks_host) *fallbacks_host = h[0];
  return SG_OK;
}
