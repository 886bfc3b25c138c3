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
//
// Two code shapes per order: SHORT (every row has <= 8 entries, e.g. the 5- and 7-point
// stencils: numpy's pairwise sum degenerates to a sequential loop) and general (8-accumulator
// blocks and the recursive split for > 129 entries, the latter out of line).
#pragma once

#include "common.cuh"

namespace sg {

enum SumOrder { kOrderNumpy = 0, kOrderSeq = 1 };

// Operand of the product val_k * X(col_k):
//   XM 0: X(j) = a[j]      XM 1: X(j) = a[j] + c b[j]      XM 2: X(j) = a[j] - c b[j]
// (XM 1/2 rebuild a vector being updated in the same pass, e.g. d' = s + beta d, without
// waiting for the update to land in memory.)
struct XF {
  const double* a;
  const double* b;
  double c;
};

template <int XM>
__device__ __forceinline__ double xval(const XF& f, int32_t j) {
  if (XM == 0) return __ldg(f.a + j);
  if (XM == 1) return add(__ldg(f.a + j), mul(f.c, __ldg(f.b + j)));
  return sub(__ldg(f.a + j), mul(f.c, __ldg(f.b + j)));
}

// Out-of-line general row reduction (long rows): plain pointer arguments only, so calling it
// does not force the caller's state through local memory.
template <int ORDER, int XM>
__device__ __noinline__ double row_general(const double* __restrict__ sv, const int32_t* __restrict__ sc,
                                           int lo, int hi, XF f) {
  auto p = [&](int64_t k) { return mul(sv[k], xval<XM>(f, sc[k])); };
  if (ORDER == kOrderSeq) return sequential_sum(p, lo, hi);
  return reduceat_sum(p, lo, hi);
}

// Row reduction over [lo, hi) of val_k * X(col_k) in ORDER.
template <int ORDER, bool SHORT, int XM>
__device__ __forceinline__ double row_reduce(const double* __restrict__ sv, const int32_t* __restrict__ sc,
                                             int lo, int hi, const XF& f) {
  if (SHORT || hi - lo <= 8) {
    if (hi <= lo) return 0.0;
    if (ORDER == kOrderSeq) {
      double s = 0.0;
      for (int k = lo; k < hi; ++k) s = add(s, mul(sv[k], xval<XM>(f, sc[k])));
      return s;
    }
    // numpy: v[lo] + pairwise(v[lo+1:hi]); pairwise of < 8 values is sequential from 0.0
    const double first = mul(sv[lo], xval<XM>(f, sc[lo]));
    if (hi - lo == 1) return first;
    double s = 0.0;
    for (int k = lo + 1; k < hi; ++k) s = add(s, mul(sv[k], xval<XM>(f, sc[k])));
    return add(first, s);
  }
  return row_general<ORDER, XM>(sv, sc, lo, hi, f);
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
template <int ORDER, bool SHORT, int XM, int ROWS, int CAP>
__device__ __forceinline__ double tile_row_dot(const RowTile<ROWS, CAP>& t, int lr,
                                               const int32_t* __restrict__ cols,
                                               const double* __restrict__ vals, const XF& f) {
  const int lo = t.offs[lr], hi = t.offs[lr + 1];
  if (t.staged) return row_reduce<ORDER, SHORT, XM>(t.vals - t.base_v, t.cols - t.base_c, lo, hi, f);
  return row_reduce<ORDER, SHORT, XM>(vals, cols, lo, hi, f);
}

}  // namespace sg
