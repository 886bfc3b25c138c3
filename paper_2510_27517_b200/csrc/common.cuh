// Shared device/host helpers for the spaigraph_b200 C-ABI library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/spaigraph_b200.h"

namespace sg {

// ------------------------------------------------------------------ error plumbing
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define SG_CUDA(call)                                         \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return ::sg::cuda_fail(_e, #call); \
  } while (0)

#define SG_LAUNCH_CHECK(what)                                   \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::sg::cuda_fail(_e, what);    \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace (ws == nullptr => size query).
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* b) : base(static_cast<char*>(b)) {}
  template <class T>
  T* take(size_t count) {
    off = align_up(off, 256);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += count * sizeof(T) + 16;
    return p;
  }
};

// ------------------------------------------------------------------ reference arithmetic
// numpy evaluates `a*b` and `a+b` as separately rounded IEEE ops; nvcc would contract them into
// DFMA.  Parity code uses these explicit round-to-nearest intrinsics instead.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) over n values produced by
// f(i), i in [0, n).  < 8: sequential from 0.0; <= 128: 8 accumulators + tree + tail;
// > 128: split at n/2 rounded down to a multiple of 8 (recursion).  SURVEY.md A.3.
template <class F>
__device__ double pairwise_leaf(const F& f, int64_t lo, int64_t n) {
  if (n < 8) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s = add(s, f(lo + i));
    return s;
  }
  double r0 = f(lo + 0), r1 = f(lo + 1), r2 = f(lo + 2), r3 = f(lo + 3);
  double r4 = f(lo + 4), r5 = f(lo + 5), r6 = f(lo + 6), r7 = f(lo + 7);
  int64_t i = 8;
  const int64_t full = n - (n % 8);
  for (; i < full; i += 8) {
    r0 = add(r0, f(lo + i + 0)); r1 = add(r1, f(lo + i + 1));
    r2 = add(r2, f(lo + i + 2)); r3 = add(r3, f(lo + i + 3));
    r4 = add(r4, f(lo + i + 4)); r5 = add(r5, f(lo + i + 5));
    r6 = add(r6, f(lo + i + 6)); r7 = add(r7, f(lo + i + 7));
  }
  double s = add(add(add(r0, r1), add(r2, r3)), add(add(r4, r5), add(r6, r7)));
  for (; i < n; ++i) s = add(s, f(lo + i));
  return s;
}

// Iterative evaluation of the recursive split (post-order with an explicit stack; depth is
// log2(n/128) <= 32 for n < 2^39).
template <class F>
__device__ double pairwise_sum(const F& f, int64_t lo, int64_t n) {
  if (n <= 128) return pairwise_leaf(f, lo, n);
  struct Frame { int64_t lo, n; double left; int state; };
  Frame st[40];
  int sp = 0;
  st[0] = {lo, n, 0.0, 0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& fr = st[sp];
    if (fr.n <= 128) {
      ret = pairwise_leaf(f, fr.lo, fr.n);
      --sp;
      continue;
    }
    int64_t n2 = fr.n / 2;
    n2 -= n2 % 8;
    if (fr.state == 0) {
      fr.state = 1;
      st[sp + 1] = {fr.lo, n2, 0.0, 0};
      ++sp;
    } else if (fr.state == 1) {
      fr.left = ret;
      fr.state = 2;
      st[sp + 1] = {fr.lo + n2, fr.n - n2, 0.0, 0};
      ++sp;
    } else {
      ret = add(fr.left, ret);
      --sp;
    }
  }
  return ret;
}

// np.add.reduceat on one nonempty segment [lo, hi): v[lo] + pairwise(v[lo+1:hi]).
template <class F>
__device__ __forceinline__ double reduceat_sum(const F& f, int64_t lo, int64_t hi) {
  if (hi <= lo) return 0.0;
  const int64_t m = hi - lo - 1;
  if (m == 0) return f(lo);
  return add(f(lo), pairwise_sum(f, lo + 1, m));
}

// np.add.at accumulation into a zero-initialised slot: ((0 + v0) + v1) + ...
template <class F>
__device__ __forceinline__ double sequential_sum(const F& f, int64_t lo, int64_t hi) {
  double s = 0.0;
  for (int64_t k = lo; k < hi; ++k) s = add(s, f(k));
  return s;
}

// ------------------------------------------------------------------ deterministic block reduce
// Fixed-shape tree (warp shuffles, then warp 0 over the per-warp partials).  Result valid in
// thread 0.  `scratch` needs blockDim.x/32 doubles.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// Two block sums sharing one pair of barriers; each value follows block_sum's tree exactly.
// Results valid in thread 0.
__device__ __forceinline__ void block_sum2(double& a, double& b) {
  __shared__ double scratch2[2][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    scratch2[0][wid] = a;
    scratch2[1][wid] = b;
  }
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  if (wid == 0) {
    a = warp_sum(lane < nw ? scratch2[0][lane] : 0.0);
    b = warp_sum(lane < nw ? scratch2[1][lane] : 0.0);
  }
}

}  // namespace sg
