// tcgen05 tensor-core path for the GNN's [edges x 24] . [24 x 24] products (SURVEY.md §8(a) a14,
// §7.2 step 5: "per-edge / per-node MLPs on tensor cores where the batched edge count makes them a
// real dense contraction").  kind::tf32 with the 3xTF32 split (a_hi b_hi + a_hi b_lo + a_lo b_hi,
// fp32 accumulation in TMEM) gives ~fp32 accuracy -- the north_star's fp32 bar is G within 1e-5.
//
// sg_tc_gemm_selftest: one 128-row tile D = A . W on the tensor core, the building block the
// fused edge pass uses; tests/test_gpu_tc.py checks it against an fp64 host product.
#include "common.cuh"
#include "tc.cuh"

namespace sg {

constexpr int kTcM = 128;  // rows per tile (one per thread of the CTA)
constexpr int kTcN = 32;   // TMEM columns / padded output width
constexpr int kTcK = 32;   // padded K

__global__ void __launch_bounds__(kTcM) k_tc_selftest(const float* __restrict__ A, const float* __restrict__ W,
                                                      int K, int N, int split3, float* __restrict__ out) {
  __shared__ __align__(128) float sAh[kTcM * kTcK];
  __shared__ __align__(128) float sAl[kTcM * kTcK];
  __shared__ __align__(128) float sBh[kTcN * kTcK];
  __shared__ __align__(128) float sBl[kTcN * kTcK];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int KP = (K + 7) / 8 * 8;
  for (int k = 0; k < KP; ++k) {
    const float a = k < K ? A[tid * K + k] : 0.f;
    const float hi = tf32_rn(a), lo = tf32_rn(a - hi);
    sAh[umma_off(tid, k, kTcM) / 4] = hi;
    sAl[umma_off(tid, k, kTcM) / 4] = lo;
  }
  for (int idx = tid; idx < kTcN * KP; idx += kTcM) {
    const int n = idx / KP, k = idx % KP;
    const float w = (n < N && k < K) ? W[k * N + n] : 0.f;
    const float hi = tf32_rn(w), lo = tf32_rn(w - hi);
    sBh[umma_off(n, k, kTcN) / 4] = hi;
    sBl[umma_off(n, k, kTcN) / 4] = lo;
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&tmem_base, kTcN);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = umma_idesc_tf32(kTcM, kTcN);
    const uint32_t a_stride = kTcM * 16, b_stride = kTcN * 16;  // bytes between K chunks (LBO)
    for (int s = 0; s < KP / 8; ++s) {
      const uint64_t ah = umma_desc(smem_u32(sAh) + 2 * s * a_stride, a_stride, 128);
      const uint64_t al = umma_desc(smem_u32(sAl) + 2 * s * a_stride, a_stride, 128);
      const uint64_t bh = umma_desc(smem_u32(sBh) + 2 * s * b_stride, b_stride, 128);
      const uint64_t bl = umma_desc(smem_u32(sBl) + 2 * s * b_stride, b_stride, 128);
      umma_tf32(taddr, ah, bh, idesc, s > 0);
      if (split3) {
        umma_tf32(taddr, ah, bl, idesc, true);
        umma_tf32(taddr, al, bh, idesc, true);
      }
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(taddr + ((uint32_t)(warp * 32) << 16), v);
#pragma unroll
  for (int n = 0; n < 32; ++n)
    if (n < N) out[tid * N + n] = v[n];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(taddr, kTcN);
}

}  // namespace sg

using namespace sg;

extern "C" int sg_tc_gemm_selftest(const float* a, const float* w, int32_t k, int32_t n, int32_t split3, float* out,
                                   void* stream) {
  if (k < 1 || k > kTcK || n < 1 || n > kTcN) { set_error("selftest: K and N must be in [1, 32]"); return SG_EINVAL; }
  k_tc_selftest<<<1, kTcM, 0, as_stream(stream)>>>(a, w, k, n, split3, out);
  SG_LAUNCH_CHECK("k_tc_selftest");
  return SG_OK;
}
