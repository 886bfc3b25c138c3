// Microbenchmark: HBM read bandwidth of a bulk-copy (cp.async.bulk + mbarrier) streaming kernel
// as a function of the number of concurrent input streams (arrays) per CTA, chunk size and
// pipeline depth -- the access pattern of the sliding-window PCG kernels without their math.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2510_27517_b200/csrc stream_bw.cu -o stream_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tma.cuh"

using namespace sg;

template <int NS, int P>
__global__ void __launch_bounds__(256, 1) k_stream(const double* const* __restrict__ arrs, long long rows_per_cta,
                                                    int C, double* out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bars[P];
  double* buf = reinterpret_cast<double*>(smraw);  // [P][NS][C]
  const long long r0 = blockIdx.x * rows_per_cta;
  const int K = (int)(rows_per_cta / C);
  auto issue = [&](int k) {
    const int ss = k % P;
    mbar_arrive_expect_tx(&bars[ss], (uint32_t)(NS * C * 8));
#pragma unroll
    for (int a = 0; a < NS; ++a) bulk_g2s(buf + (ss * NS + a) * C, arrs[a] + r0 + (long long)k * C, C * 8, &bars[ss]);
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < P; ++q) mbar_init(&bars[q], 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < P - 1 && k < K; ++k) issue(k);
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    mbar_wait(&bars[k % P], (uint32_t)((k / P) & 1));
    for (int a = 0; a < NS; ++a)
      for (int i = threadIdx.x; i < C; i += 256) acc += buf[((k % P) * NS + a) * C + i];
    __syncthreads();
    if (threadIdx.x == 0 && k + P - 1 < K) issue(k + P - 1);
  }
  if (acc == 12345.0) out[0] = acc;
}

template <int NS, int P>
void run(double** d_arrs, long long n, int ctas_per_sm, int C) {
  const int sms = 148;
  const int grid = sms * ctas_per_sm;
  const long long rows = n / grid / C * C;
  const size_t smem = (size_t)P * NS * C * 8;
  cudaFuncSetAttribute(k_stream<NS, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double** dptr;
  cudaMalloc(&dptr, NS * sizeof(double*));
  cudaMemcpy(dptr, d_arrs, NS * sizeof(double*), cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k_stream<NS, P><<<grid, 256, smem>>>((const double* const*)dptr, rows, C, out);
  cudaEventRecord(e0);
  const int it = 5;
  for (int w = 0; w < it; ++w) k_stream<NS, P><<<grid, 256, smem>>>((const double* const*)dptr, rows, C, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)NS * rows * grid * 8 * it;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stream<NS, P>, 256, smem);
  printf("streams %2d  P %d  chunk %4d rows  CTAs/SM %d (occ %d)  smem %6zu B  ->  %7.1f GB/s  (%s)\n", NS, P, C,
         ctas_per_sm, occ, smem, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(dptr);
  cudaFree(out);
}


// One interleaved block of NB "diagonals" per chunk (a single NB*C*8-byte copy from a
// [chunk][NB][C] layout) + NS separate vector streams: TMA (VT = 1) or plain loads (VT = 0).
template <int NB, int NS, int P, int VT>
__global__ void __launch_bounds__(256, 1) k_mixed(const double* __restrict__ blk, const double* const* __restrict__ arrs,
                                                   long long rows_per_cta, int C, double* out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bars[P];
  double* buf = reinterpret_cast<double*>(smraw);  // [P][NB + NS][C]
  const long long r0 = blockIdx.x * rows_per_cta;
  const int K = (int)(rows_per_cta / C);
  auto issue = [&](int k) {
    const int ss = k % P;
    mbar_arrive_expect_tx(&bars[ss], (uint32_t)((NB + (VT ? NS : 0)) * C * 8));
    bulk_g2s(buf + (ss * (NB + NS)) * C, blk + (r0 + (long long)k * C) * NB, NB * C * 8, &bars[ss]);
    if (VT)
#pragma unroll
      for (int a = 0; a < NS; ++a)
        bulk_g2s(buf + (ss * (NB + NS) + NB + a) * C, arrs[a] + r0 + (long long)k * C, C * 8, &bars[ss]);
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < P; ++q) mbar_init(&bars[q], 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < P - 1 && k < K; ++k) issue(k);
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    double v[NS > 0 ? NS : 1];
    if (!VT)
#pragma unroll
      for (int a = 0; a < NS; ++a) v[a] = __ldg(arrs[a] + r0 + (long long)k * C + threadIdx.x);
    mbar_wait(&bars[k % P], (uint32_t)((k / P) & 1));
    for (int a = 0; a < NB + (VT ? NS : 0); ++a)
      for (int i = threadIdx.x; i < C; i += 256) acc += buf[((k % P) * (NB + NS) + a) * C + i];
    if (!VT)
#pragma unroll
      for (int a = 0; a < NS; ++a) acc += v[a];
    __syncthreads();
    if (threadIdx.x == 0 && k + P - 1 < K) issue(k + P - 1);
  }
  if (acc == 12345.0) out[0] = acc;
}

template <int NB, int NS, int P, int VT>
void run_mixed(double* blk, double** d_arrs, long long n, int ctas_per_sm, int C) {
  const int grid = 148 * ctas_per_sm;
  const long long rows = n / grid / C * C;
  const size_t smem = (size_t)P * (NB + NS) * C * 8;
  cudaFuncSetAttribute(k_mixed<NB, NS, P, VT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double** dptr;
  cudaMalloc(&dptr, 16 * sizeof(double*));
  cudaMemcpy(dptr, d_arrs, 16 * sizeof(double*), cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k_mixed<NB, NS, P, VT><<<grid, 256, smem>>>(blk, (const double* const*)dptr, rows, C, out);
  cudaEventRecord(e0);
  const int it = 5;
  for (int w = 0; w < it; ++w) k_mixed<NB, NS, P, VT><<<grid, 256, smem>>>(blk, (const double* const*)dptr, rows, C, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)(NB + NS) * rows * grid * 8 * it;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mixed<NB, NS, P, VT>, 256, smem);
  printf("block %d diag + %d vectors (%s)  P %d  chunk %4d  CTAs/SM %d (occ %d)  smem %6zu  ->  %7.1f GB/s  (%s)\n", NB, NS,
         VT ? "bulk" : "ld", P, C, ctas_per_sm, occ, smem, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(dptr);
  cudaFree(out);
}

int main() {
  const long long n = 1LL << 26;  // 64 Mi rows per array = 512 MB
  double* arrs[16];
  for (int a = 0; a < 16; ++a) {
    cudaMalloc(&arrs[a], n * 8);
    cudaMemset(arrs[a], 0, n * 8);
  }
  double* blk;
  cudaMalloc(&blk, 5 * n * 8);
  cudaMemset(blk, 0, 5 * n * 8);
  // separate 2 KB streams (the sliding-window / strip kernels' layout): streams x depth x CTAs/SM
  run<2, 3>(arrs, n, 3, 256);
  run<4, 3>(arrs, n, 3, 256);
  run<8, 3>(arrs, n, 3, 256);
  run<10, 2>(arrs, n, 3, 256);
  run<10, 3>(arrs, n, 2, 256);
  run<10, 4>(arrs, n, 2, 256);
  run<4, 6>(arrs, n, 4, 256);
  run<4, 8>(arrs, n, 3, 256);
  // larger copies
  run<10, 2>(arrs, n, 1, 1024);
  run<4, 3>(arrs, n, 2, 1024);
  run<8, 3>(arrs, n, 3, 512);
  run<8, 3>(arrs, n, 2, 512);
  run<4, 3>(arrs, n, 3, 1024);
  run<2, 3>(arrs, n, 3, 2048);
  // 5 diagonals as one interleaved block copy per chunk + vector streams (bulk or plain loads)
  run_mixed<5, 4, 2, 1>(blk, arrs, n, 3, 256);
  run_mixed<5, 4, 3, 1>(blk, arrs, n, 3, 256);
  run_mixed<5, 4, 3, 0>(blk, arrs, n, 3, 256);
  run_mixed<5, 2, 3, 1>(blk, arrs, n, 3, 256);
  run_mixed<5, 2, 3, 0>(blk, arrs, n, 3, 256);
  run_mixed<5, 0, 3, 1>(blk, arrs, n, 3, 256);
  run_mixed<3, 2, 4, 1>(blk, arrs, n, 4, 256);
  run_mixed<3, 2, 4, 0>(blk, arrs, n, 4, 256);
  return 0;
}
