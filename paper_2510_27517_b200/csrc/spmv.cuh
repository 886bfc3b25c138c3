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

// ------------------------------------------------------------------ warp per row, numpy order
// np.add.reduceat of one long row [lo, hi), evaluated by a whole warp yet bit-identical to
// reduceat_sum: v[lo] + pairwise(m = hi - lo - 1 values).  numpy's pairwise recursion splits
// m > 128 into LEAVES of 64..128 values (left to right); each leaf sums 8 stride-8 accumulators
// sequentially, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then its m % 8 tail in order.  Here the
// 8 accumulators of a leaf are 8 lanes (4 leaves per pass, each lane walking its accumulator's
// stride-8 subsequence in the same order, 8 consecutive values per 8 lanes => coalesced), the
// accumulator tree is a 3-level xor butterfly (IEEE a + b == b + a bitwise, so the pairing is the
// reference's), the tail is added by the leaf's first lane, and lane 0 combines the leaf sums
// along the recursion.  Leaf table and sums live in the caller's per-warp shared scratch.
// m > kWarpMaxVals (more than 32 leaves) falls back to lane 0 walking the row alone.
constexpr int kWarpLeaves = 32;
constexpr int kWarpMaxVals = 64 * kWarpLeaves;

template <int XM>
__device__ __noinline__ double warp_row_numpy(const double* __restrict__ vals, const int32_t* __restrict__ cols,
                                              int lo, int hi, XF f, int2* __restrict__ leaf,
                                              double* __restrict__ lsum) {
  const int lane = threadIdx.x & 31;
  auto p = [&](int k) { return mul(__ldg(vals + k), xval<XM>(f, __ldg(cols + k))); };
  if (hi <= lo) return 0.0;
  const int m = hi - lo - 1;
  double res = 0.0;
  if (m < 8 || m > kWarpMaxVals) {
    if (lane == 0) res = reduceat_sum(p, lo, hi);
    return __shfl_sync(0xffffffffu, res, 0);
  }
  int nl = 0;
  if (lane == 0) {  // leaves of the recursion, left to right (depth <= log2(2048 / 64) + 1)
    int2 stk[8];
    int sp = 0;
    stk[0] = make_int2(0, m);
    while (sp >= 0) {
      const int2 fr = stk[sp--];
      if (fr.y <= 128) {
        leaf[nl++] = fr;
      } else {
        int n2 = fr.y / 2;
        n2 -= n2 % 8;
        stk[++sp] = make_int2(fr.x + n2, fr.y - n2);
        stk[++sp] = make_int2(fr.x, n2);
      }
    }
  }
  nl = __shfl_sync(0xffffffffu, nl, 0);
  __syncwarp();
  const int j = lane & 7;
  const int base0 = lo + 1;
  for (int g0 = 0; g0 < nl; g0 += 4) {
    const int li = g0 + (lane >> 3);
    double r = 0.0;
    int2 L = make_int2(0, 0);
    if (li < nl) {
      L = leaf[li];
      const int b = base0 + L.x, full = L.y & ~7;
      r = p(b + j);
      int i = j + 8;
      for (; i + 24 < full; i += 32) {
        const double v0 = p(b + i), v1 = p(b + i + 8), v2 = p(b + i + 16), v3 = p(b + i + 24);
        r = add(add(add(add(r, v0), v1), v2), v3);
      }
      for (; i < full; i += 8) r = add(r, p(b + i));
    }
    r = add(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = add(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = add(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (li < nl && j == 0) {
      const int b = base0 + L.x;
      for (int i = L.y & ~7; i < L.y; ++i) r = add(r, p(b + i));
      lsum[li] = r;
    }
  }
  __syncwarp();
  if (lane == 0) {  // post-order combine along the same recursion
    struct Fr { int n, state; double left; };
    Fr st[8];
    int sp = 0, next = 0;
    st[0] = {m, 0, 0.0};
    double ret = 0.0;
    while (sp >= 0) {
      Fr& fr = st[sp];
      if (fr.n <= 128) { ret = lsum[next++]; --sp; continue; }
      int n2 = fr.n / 2;
      n2 -= n2 % 8;
      if (fr.state == 0) { fr.state = 1; st[++sp] = {n2, 0, 0.0}; }
      else if (fr.state == 1) { fr.left = ret; fr.state = 2; st[++sp] = {fr.n - n2, 0, 0.0}; }
      else { ret = add(fr.left, ret); --sp; }
    }
    res = add(p(lo), ret);
  }
  __syncwarp();
  return __shfl_sync(0xffffffffu, res, 0);
}

}  // namespace sg
