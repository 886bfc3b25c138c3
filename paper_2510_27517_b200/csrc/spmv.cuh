// CSR row-block machinery shared by the SpMV, PCG and loss kernels.
//
// Layout in HBM: int32 row offsets, int32 column indices, f64 values (CSR, the reference's
// storage order).  A CTA owns ROWS consecutive rows.  It first streams the rows' nonzeros
// (values + column indices, one contiguous byte range) into shared memory with 16-byte vector
// loads — fully coalesced regardless of row lengths ("CSR-stream") — then each thread reduces
// one row from shared memory in the reference's summation order:
//   kOrderNumpy: np.add.reduceat order, v[lo] + pairwise(v[lo+1:hi])   (spmv, sparse.py:186)
//   kOrderSeq:   ((0 + v0) + v1) + ...  == np.add.at into zeros          (spmv_transpose, :194)
// Products are rounded before summation (no FMA), so results are bit-identical to numpy.
// Blocks whose nonzeros exceed the shared-memory capacity fall back to direct global loads.
#pragma once

#include "common.cuh"

namespace sg {

enum SumOrder { kOrderNumpy = 0, kOrderSeq = 1 };

template <class F>
__device__ __noinline__ double pairwise_long(const F& f, int64_t lo, int64_t n) {
  return pairwise_sum(f, lo, n);
}

// Row reduction over entries [lo, hi) of a product functor p(k), in the requested order.
template <int ORDER, class P>
__device__ __forceinline__ double row_reduce(const P& p, int lo, int hi) {
  if (ORDER == kOrderSeq) {
    double s = 0.0;
    for (int k = lo; k < hi; ++k) s = add(s, p(k));
    return s;
  }
  if (hi <= lo) return 0.0;
  const int m = hi - lo - 1;
  const double first = p(lo);
  if (m == 0) return first;
  if (m <= 128) return add(first, pairwise_leaf(p, (int64_t)lo + 1, (int64_t)m));
  return add(first, pairwise_long(p, (int64_t)lo + 1, (int64_t)m));
}

// Shared-memory tile of one CTA's rows.
template <int ROWS, int CAP>
struct __align__(16) RowTile {
  static_assert(CAP % 4 == 0, "CAP must be a multiple of 4");
  double vals[CAP + 2];
  int32_t cols[CAP + 4];
  int32_t offs[ROWS + 1];
  int base_v, base_c;  // first staged element index (aligned down) for vals / cols
  int staged;          // 1 if the tile holds the nonzeros, 0 => direct global reads
};

// Stage rows [r0, r1) of (offs, cols, vals).  All threads participate; ends with a barrier.
template <int ROWS, int CAP>
__device__ __forceinline__ void stage_rows(RowTile<ROWS, CAP>& t, int64_t r0, int64_t r1,
                                           const int32_t* __restrict__ offs,
                                           const int32_t* __restrict__ cols,
                                           const double* __restrict__ vals) {
  const int nr = (int)(r1 - r0);
  for (int i = threadIdx.x; i <= nr; i += blockDim.x) t.offs[i] = __ldg(offs + r0 + i);
  __syncthreads();
  const int e0 = t.offs[0], e1 = t.offs[nr];
  const int a0v = e0 & ~1, a1v = (e1 + 1) & ~1;
  const int a0c = e0 & ~3, a1c = (e1 + 3) & ~3;
  const bool fits = (a1v - a0v) <= CAP + 2 && (a1c - a0c) <= CAP + 4;
  if (fits) {
    const double2* sv = reinterpret_cast<const double2*>(vals + a0v);
    double2* dv = reinterpret_cast<double2*>(t.vals);
    const int nv = (a1v - a0v) >> 1;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) dv[i] = __ldg(sv + i);
    const int4* sc = reinterpret_cast<const int4*>(cols + a0c);
    int4* dc = reinterpret_cast<int4*>(t.cols);
    const int nc = (a1c - a0c) >> 2;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) dc[i] = __ldg(sc + i);
  }
  if (threadIdx.x == 0) {
    t.base_v = a0v;
    t.base_c = a0c;
    t.staged = fits ? 1 : 0;
  }
  __syncthreads();
}

// y_i = sum_k val_k * X(col_k) for local row `lr` of a staged tile, in ORDER.
template <int ORDER, int ROWS, int CAP, class XF>
__device__ __forceinline__ double tile_row_dot(const RowTile<ROWS, CAP>& t, int lr,
                                               const int32_t* __restrict__ cols,
                                               const double* __restrict__ vals, const XF& xf) {
  const int lo = t.offs[lr], hi = t.offs[lr + 1];
  if (t.staged) {
    const double* sv = t.vals - t.base_v;
    const int32_t* sc = t.cols - t.base_c;
    return row_reduce<ORDER>([&](int64_t k) { return mul(sv[k], xf(sc[k])); }, lo, hi);
  }
  return row_reduce<ORDER>([&](int64_t k) { return mul(__ldg(vals + k), xf(__ldg(cols + k))); }, lo, hi);
}

}  // namespace sg
