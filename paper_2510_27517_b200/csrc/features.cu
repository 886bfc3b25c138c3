// Norms, graph features and stencil generators.
//
// sg_matrix_norm reproduces math.fsum exactly: every |v| (or fl(v*v)) is added as an integer
// into a 2100-bit fixed-point superaccumulator (32-bit limbs held in uint64; integer atomics
// make the result independent of thread order), then rounded once, round-half-even.  That is
// the correctly rounded sum fsum promises, so `norm_A` is bit-identical to the reference.
#include "common.cuh"

namespace sg {

constexpr int NLIMB = 72;  // 72*32 = 2304 bits >= 2098 value bits + carry headroom

// Add an integer mantissa sum `m` (< 2^63) whose least significant bit sits at fixed-point
// position g0 (one limb = 32 bits).
__device__ __forceinline__ void accum_add_int(unsigned long long* limbs, unsigned long long m, int g0) {
  const int L = g0 >> 5, s = g0 & 31;
  const unsigned long long lo = m << s;
  const unsigned long long hi = s ? (m >> (64 - s)) : 0ull;
  atomicAdd(&limbs[L], lo & 0xFFFFFFFFull);
  atomicAdd(&limbs[L + 1], lo >> 32);
  if (hi) atomicAdd(&limbs[L + 2], hi);
}

// Segmented exact accumulation: blockIdx.y = segment (system), blockIdx.x strides over it.
// Lanes holding values with the same binary exponent first sum their mantissas as integers
// (__match_any_sync: <= 32 x 2^53 < 2^58, exact), so one shared-memory atomic triple is issued
// per distinct exponent per warp instead of per value.
// mode 0: |v|, mode 1: fl(v*v).  flags: bit0 inf, bit1 nan.
__global__ void k_exact_accum(const double* __restrict__ v, const int64_t* __restrict__ seg, int mode,
                              unsigned long long* g_limbs, unsigned int* flags) {
  __shared__ unsigned long long sl[NLIMB];
  for (int i = threadIdx.x; i < NLIMB; i += blockDim.x) sl[i] = 0;
  __syncthreads();
  const int sg = blockIdx.y;
  const int64_t lo = seg[sg], hi = seg[sg + 1];
  unsigned int f = 0;
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count so that every lane takes part in __match_any_sync
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t base = lo + (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
  for (int64_t kb = base; kb < hi; kb += stride) {
    const int64_t k = kb + lane;
    int key = -1;  // -1: no contribution
    unsigned long long m = 0;
    if (k < hi) {
      const double x = v[k];
      const double a = mode == 1 ? mul(x, x) : fabs(x);
      if (isnan(a)) f |= 2;
      else if (isinf(a)) f |= 1;
      else {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(a);
        const int ex = (int)((bits >> 52) & 0x7FF);
        m = bits & ((1ull << 52) - 1);
        if (ex) m |= (1ull << 52);
        if (m) key = ex ? ex - 1 : 0;  // fixed-point position of the mantissa's lsb
      }
    }
    const unsigned int peers = __match_any_sync(0xffffffffu, key);
    // each lane sums the mantissas of its group (exact integer arithmetic, uniform shuffles)
    unsigned long long gsum = 0;
#pragma unroll 4
    for (int src = 0; src < 32; ++src) {
      const unsigned long long ms = __shfl_sync(0xffffffffu, m, src);
      if ((peers >> src) & 1u) gsum += ms;
    }
    if (key >= 0 && lane == __ffs(peers) - 1) accum_add_int(sl, gsum, key);
  }
  if (f) atomicOr(&flags[sg], f);
  __syncthreads();
  for (int i = threadIdx.x; i < NLIMB; i += blockDim.x)
    if (sl[i]) atomicAdd(&g_limbs[(int64_t)sg * NLIMB + i], sl[i]);
}

__device__ double round_limbs(const unsigned long long* in) {
  unsigned int l[NLIMB];
  unsigned long long c = 0;
  for (int i = 0; i < NLIMB; ++i) {
    unsigned long long t = in[i] + c;
    l[i] = (unsigned int)(t & 0xFFFFFFFFull);
    c = t >> 32;
  }
  int top = -1;
  for (int i = NLIMB - 1; i >= 0; --i)
    if (l[i]) { top = i; break; }
  if (top < 0) return 0.0;
  const int P = 32 * top + (31 - __clz(l[top]));
  auto bit = [&](int i) -> unsigned long long { return (l[i >> 5] >> (i & 31)) & 1u; };
  if (P <= 52) {
    unsigned long long iv = (unsigned long long)l[0] | ((unsigned long long)l[1] << 32);
    return ldexp((double)iv, -1074);
  }
  int shift = P - 52;
  unsigned long long mant = 0;
  for (int i = P; i >= shift; --i) mant = (mant << 1) | bit(i);
  const unsigned long long rbit = bit(shift - 1);
  bool sticky = false;
  for (int i = 0; i < shift - 1 && !sticky; ++i) {
    if ((i & 31) == 0 && i + 32 <= shift - 1) {
      if (l[i >> 5]) sticky = true;
      i += 31;
      continue;
    }
    if (bit(i)) sticky = true;
  }
  if (rbit && (sticky || (mant & 1))) {
    ++mant;
    if (mant == (1ull << 53)) { mant >>= 1; ++shift; }
  }
  return ldexp((double)mant, shift - 1074);
}

// One block per segment (thread 0 works): round the segment's limbs once, apply the kind.
__global__ void k_norm_finish(const unsigned long long* limbs, const unsigned int* flags,
                              const int64_t* __restrict__ seg, int kind, double* out) {
  if (threadIdx.x != 0) return;
  const int sg = blockIdx.x;
  const int64_t nnz = seg[sg + 1] - seg[sg];
  double s;
  if (flags[sg] & 2) s = __longlong_as_double(0x7ff8000000000000ll);
  else if (flags[sg] & 1) s = __longlong_as_double(0x7ff0000000000000ll);
  else s = round_limbs(limbs + (int64_t)sg * NLIMB);
  if (kind == 0) s = __ddiv_rn(s, (double)nnz);
  else if (kind == 1) s = __dsqrt_rn(s);
  out[sg] = s;
}

// graphfeat.py:83 and 93-104, for rows row0 .. row0+n-1 (local index li = i - row0) that are rows
// grow0 + li of a matrix with n_global rows (grid coordinates and rowsum / n use the global
// matrix: a row partition's block of rows gets exactly the global features).
__global__ void k_graph_features(int64_t n, int64_t row0, int64_t grow0, int64_t n_global,
                                 const int32_t* __restrict__ offs,
                                 const int32_t* __restrict__ cols, const double* __restrict__ vals,
                                 const double* __restrict__ norm_p, int family, int64_t nx,
                                 int64_t ny, const double* __restrict__ coeff, double coeff_mean,
                                 double* node_out, double* edge_out) {
  const double norm = *norm_p;
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < n;
       li += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = row0 + li;
    const int32_t lo = offs[i], hi = offs[i + 1];
    for (int32_t k = lo; k < hi; ++k) edge_out[k] = __ddiv_rn(vals[k], norm);
    if (family == 1) {
      const double hx = __ddiv_rn(1.0, (double)(nx + 1)), hy = __ddiv_rn(1.0, (double)(ny + 1));
      const int64_t ix = (grow0 + li) % nx, iy = (grow0 + li) / nx;
      node_out[3 * i + 0] = mul((double)(ix + 1), hx);
      node_out[3 * i + 1] = mul((double)(iy + 1), hy);
      node_out[3 * i + 2] = __ddiv_rn(coeff[li], coeff_mean);
    } else {
      double rs = reduceat_sum([&](int64_t k) { return vals[k]; }, lo, hi);
      double dg = 0.0;
      for (int32_t k = lo; k < hi; ++k)
        if (cols[k] == (int32_t)i) dg = vals[k];
      node_out[2 * i + 0] = __ddiv_rn(__ddiv_rn(rs, (double)n_global), norm);
      node_out[2 * i + 1] = __ddiv_rn(dg, norm);
    }
  }
}

// Exact-sum accumulator in transferable form: carries propagated (every limb < 2^32) plus the
// inf / nan counts, so accumulators of several row blocks (ranks) can be added limb by limb.
__global__ void k_norm_export(const unsigned long long* limbs, const unsigned int* flags, unsigned long long* acc) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long c = 0;
  for (int i = 0; i < NLIMB; ++i) {
    const unsigned long long t = limbs[i] + c;
    acc[i] = t & 0xFFFFFFFFull;
    c = t >> 32;
  }
  acc[NLIMB - 1] += c << 32;  // never reached for finite doubles (2304 bits of headroom)
  acc[NLIMB] = (flags[0] & 1u) ? 1ull : 0ull;
  acc[NLIMB + 1] = (flags[0] & 2u) ? 1ull : 0ull;
}

__global__ void k_norm_import(const unsigned long long* acc, int64_t count, int kind, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s;
  if (acc[NLIMB + 1]) s = __longlong_as_double(0x7ff8000000000000ll);
  else if (acc[NLIMB]) s = __longlong_as_double(0x7ff0000000000000ll);
  else s = round_limbs(acc);
  if (kind == 0) s = __ddiv_rn(s, (double)count);
  else if (kind == 1) s = __dsqrt_rn(s);
  *out = s;
}

// Batched features: every row of a block-diagonal batch, system found by binary search.
__global__ void k_graph_features_batched(const int64_t* __restrict__ row_start, int n_sys, int64_t n,
                                         const int32_t* __restrict__ offs, const int32_t* __restrict__ cols,
                                         const double* __restrict__ vals, const double* __restrict__ norms,
                                         int family, const int64_t* __restrict__ nx_arr,
                                         const int64_t* __restrict__ ny_arr, const double* __restrict__ coeff,
                                         const double* __restrict__ coeff_mean, double* node_out,
                                         double* edge_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_sys;  // largest sg with row_start[sg] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (row_start[mid] <= i) lo = mid; else hi = mid;
    }
    const int sg = lo;
    const int64_t r0 = row_start[sg], ns = row_start[sg + 1] - r0, li = i - r0;
    const double norm = norms[sg];
    const int32_t e0 = offs[i], e1 = offs[i + 1];
    for (int32_t k = e0; k < e1; ++k) edge_out[k] = __ddiv_rn(vals[k], norm);
    if (family == 1) {
      const int64_t nx = nx_arr[sg], ny = ny_arr[sg];
      const double hx = __ddiv_rn(1.0, (double)(nx + 1)), hy = __ddiv_rn(1.0, (double)(ny + 1));
      node_out[3 * i + 0] = mul((double)(li % nx + 1), hx);
      node_out[3 * i + 1] = mul((double)(li / nx + 1), hy);
      node_out[3 * i + 2] = __ddiv_rn(coeff[i], coeff_mean[sg]);
    } else {
      const double rs = reduceat_sum([&](int64_t k) { return vals[k]; }, e0, e1);
      double dg = 0.0;
      for (int32_t k = e0; k < e1; ++k)
        if (cols[k] == (int32_t)i) dg = vals[k];
      node_out[2 * i + 0] = __ddiv_rn(__ddiv_rn(rs, (double)ns), norm);
      node_out[2 * i + 1] = __ddiv_rn(dg, norm);
    }
  }
}

// ------------------------------------------------------------------ stencil generators
// Entries stored before node (ix, iy) of the 5-point grid, rows in idx = ix + nx*iy order.
__device__ __forceinline__ int64_t before2d(int64_t ix, int64_t iy, int64_t nx, int64_t ny) {
  int64_t full = iy * (3 * nx - 2) + nx * (iy > 0 ? iy - 1 : 0) + nx * (iy < ny - 1 ? iy : ny - 1);
  int64_t per = 1 + (iy > 0) + (iy < ny - 1);
  int64_t part = ix * per + (ix > 0 ? ix - 1 : 0) + (ix < nx - 1 ? ix : nx - 1);
  return full + part;
}

// datasets.py:108-143 (face means, 1/h^2 scaling, boundary faces keep the node's value).
__global__ void k_poisson2d(int64_t nx, int64_t ny, const double* __restrict__ a, int64_t row0,
                            int64_t nnz0, int32_t* offs, int32_t* cols, double* vals) {
  const int64_t n = nx * ny;
  const double ihx2 = (double)((nx + 1) * (nx + 1)), ihy2 = (double)((ny + 1) * (ny + 1));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { offs[row0 + n] = (int32_t)(nnz0 + 5 * n - 2 * nx - 2 * ny); continue; }
    const int64_t ix = i % nx, iy = i / nx;
    const double c = a[i];
    const double w = ix > 0 ? mul(0.5, add(c, a[i - 1])) : c;
    const double e = ix < nx - 1 ? mul(0.5, add(c, a[i + 1])) : c;
    const double s = iy > 0 ? mul(0.5, add(c, a[i - nx])) : c;
    const double nn = iy < ny - 1 ? mul(0.5, add(c, a[i + nx])) : c;
    int64_t k = nnz0 + before2d(ix, iy, nx, ny);
    const int64_t gi = row0 + i;
    offs[gi] = (int32_t)k;
    if (iy > 0) { cols[k] = (int32_t)(gi - nx); vals[k] = mul(-s, ihy2); ++k; }
    if (ix > 0) { cols[k] = (int32_t)(gi - 1); vals[k] = mul(-w, ihx2); ++k; }
    cols[k] = (int32_t)gi; vals[k] = add(mul(add(w, e), ihx2), mul(add(s, nn), ihy2)); ++k;
    if (ix < nx - 1) { cols[k] = (int32_t)(gi + 1); vals[k] = mul(-e, ihx2); ++k; }
    if (iy < ny - 1) { cols[k] = (int32_t)(gi + nx); vals[k] = mul(-nn, ihy2); ++k; }
  }
}

__device__ __forceinline__ int64_t before3d(int64_t ix, int64_t iy, int64_t iz, int64_t nx,
                                            int64_t ny, int64_t nz) {
  const int64_t plane = nx * ny + 2 * (nx - 1) * ny + 2 * nx * (ny - 1);
  const int64_t nxy = nx * ny;
  int64_t full = iz * plane + nxy * (iz > 0 ? iz - 1 : 0) + nxy * (iz < nz - 1 ? iz : nz - 1);
  const int64_t zc = (iz > 0) + (iz < nz - 1);
  int64_t rows = iy * (3 * nx - 2) + nx * (iy > 0 ? iy - 1 : 0) + nx * (iy < ny - 1 ? iy : ny - 1) +
                 iy * nx * zc;
  const int64_t per = 1 + (iy > 0) + (iy < ny - 1) + zc;
  int64_t part = ix * per + (ix > 0 ? ix - 1 : 0) + (ix < nx - 1 ? ix : nx - 1);
  return full + rows + part;
}

__global__ void k_poisson3d(int64_t nx, int64_t ny, int64_t nz, int32_t* offs, int32_t* cols,
                            double* vals) {
  const int64_t nxy = nx * ny, n = nxy * nz;
  const double ihx2 = (double)((nx + 1) * (nx + 1)), ihy2 = (double)((ny + 1) * (ny + 1)),
               ihz2 = (double)((nz + 1) * (nz + 1));
  const double dv = add(add(mul(2.0, ihx2), mul(2.0, ihy2)), mul(2.0, ihz2));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { offs[n] = (int32_t)(7 * n - 2 * (nxy * nz / nx) - 2 * (nxy * nz / ny) - 2 * nxy); continue; }
    const int64_t ix = i % nx, iy = (i / nx) % ny, iz = i / nxy;
    int64_t k = before3d(ix, iy, iz, nx, ny, nz);
    offs[i] = (int32_t)k;
    if (iz > 0) { cols[k] = (int32_t)(i - nxy); vals[k] = -ihz2; ++k; }
    if (iy > 0) { cols[k] = (int32_t)(i - nx); vals[k] = -ihy2; ++k; }
    if (ix > 0) { cols[k] = (int32_t)(i - 1); vals[k] = -ihx2; ++k; }
    cols[k] = (int32_t)i; vals[k] = dv; ++k;
    if (ix < nx - 1) { cols[k] = (int32_t)(i + 1); vals[k] = -ihx2; ++k; }
    if (iy < ny - 1) { cols[k] = (int32_t)(i + nx); vals[k] = -ihy2; ++k; }
    if (iz < nz - 1) { cols[k] = (int32_t)(i + nxy); vals[k] = -ihz2; ++k; }
  }
}

static inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = ceil_div(n > 0 ? n : 1, threads);
  return (int)(g > 148 * 32 ? 148 * 32 : g);
}

}  // namespace sg

using namespace sg;

static int norm_segments(const double* vals, const int64_t* seg_dev, int32_t n_seg, int64_t max_len, int kind,
                         double* out, unsigned long long* limbs, unsigned int* flags, cudaStream_t s) {
  if (kind < 0 || kind > 2) { set_error("unknown norm kind"); return SG_EINVAL; }
  SG_CUDA(cudaMemsetAsync(limbs, 0, (size_t)n_seg * NLIMB * sizeof(unsigned long long), s));
  SG_CUDA(cudaMemsetAsync(flags, 0, (size_t)n_seg * sizeof(unsigned int), s));
  int bx = (int)ceil_div(max_len > 0 ? max_len : 1, 256);
  const int cap = (int)ceil_div(148 * 16, n_seg);
  if (bx > cap) bx = cap < 1 ? 1 : cap;
  k_exact_accum<<<dim3(bx, n_seg), 256, 0, s>>>(vals, seg_dev, kind == 1 ? 1 : 0, limbs, flags);
  SG_LAUNCH_CHECK("k_exact_accum");
  k_norm_finish<<<n_seg, 32, 0, s>>>(limbs, flags, seg_dev, kind, out);
  SG_LAUNCH_CHECK("k_norm_finish");
  return SG_OK;
}

extern "C" int sg_matrix_norm(const double* vals, int64_t nnz, int kind, double* norm_out,
                              void* ws, size_t* ws_bytes, void* stream) {
  Carve c(ws);
  unsigned long long* limbs = c.take<unsigned long long>(NLIMB);
  unsigned int* flags = c.take<unsigned int>(1);
  int64_t* seg = c.take<int64_t>(2);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (nnz <= 0) { set_error("norm of a matrix with no stored entries"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  const int64_t h[2] = {0, nnz};
  SG_CUDA(cudaMemcpyAsync(seg, h, sizeof(h), cudaMemcpyHostToDevice, s));
  return norm_segments(vals, seg, 1, nnz, kind, norm_out, limbs, flags, s);
}

extern "C" int sg_matrix_norm_batched(const double* vals, const int64_t* seg_start, int32_t n_seg,
                                      int64_t max_seg_len, int kind, double* norms_out, void* ws,
                                      size_t* ws_bytes, void* stream) {
  Carve c(ws);
  unsigned long long* limbs = c.take<unsigned long long>((size_t)(n_seg > 0 ? n_seg : 1) * NLIMB);
  unsigned int* flags = c.take<unsigned int>(n_seg > 0 ? n_seg : 1);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (n_seg <= 0) return SG_OK;
  return norm_segments(vals, seg_start, n_seg, max_seg_len, kind, norms_out, limbs, flags, as_stream(stream));
}

extern "C" int sg_graph_features(int64_t n, int64_t row0, const int32_t* offs, const int32_t* cols,
                                 const double* vals, const double* norm, int family, int64_t nx,
                                 int64_t ny, const double* coeff, double coeff_mean,
                                 double* node_out, double* edge_out, void* stream) {
  if (family == 1 && nx * ny != n) { set_error("meta grid does not match matrix size"); return SG_EINVAL; }
  if (n <= 0) return SG_OK;
  k_graph_features<<<grid_for(n), 256, 0, as_stream(stream)>>>(n, row0, 0, n, offs, cols, vals, norm, family,
                                                               nx, ny, coeff, coeff_mean,
                                                               node_out, edge_out);
  SG_LAUNCH_CHECK("k_graph_features");
  return SG_OK;
}

extern "C" int sg_graph_features_batched(const int64_t* row_start, int32_t n_sys, int64_t n, const int32_t* offs,
                                         const int32_t* cols, const double* vals, const double* norms, int family,
                                         const int64_t* nx, const int64_t* ny, const double* coeff,
                                         const double* coeff_mean, double* node_out, double* edge_out,
                                         void* stream) {
  if (n <= 0 || n_sys <= 0) return SG_OK;
  k_graph_features_batched<<<grid_for(n), 256, 0, as_stream(stream)>>>(row_start, n_sys, n, offs, cols, vals, norms,
                                                                      family, nx, ny, coeff, coeff_mean, node_out,
                                                                      edge_out);
  SG_LAUNCH_CHECK("k_graph_features_batched");
  return SG_OK;
}

extern "C" int sg_gen_poisson2d(int64_t nx, int64_t ny, const double* coeff, int64_t row0,
                                int64_t nnz0, int32_t* offs, int32_t* cols, double* vals,
                                void* stream) {
  if (nx < 1 || ny < 1) { set_error("grid dimensions must be positive"); return SG_EINVAL; }
  if (nnz0 + 5 * nx * ny >= (int64_t)INT32_MAX || row0 + nx * ny >= (int64_t)INT32_MAX) {
    set_error("grid too large for int32 indices");
    return SG_EINVAL;
  }
  k_poisson2d<<<grid_for(nx * ny + 1), 256, 0, as_stream(stream)>>>(nx, ny, coeff, row0, nnz0, offs, cols, vals);
  SG_LAUNCH_CHECK("k_poisson2d");
  return SG_OK;
}

extern "C" int sg_gen_poisson3d(int64_t nx, int64_t ny, int64_t nz, int32_t* offs, int32_t* cols,
                                double* vals, void* stream) {
  if (nx < 1 || ny < 1 || nz < 1) { set_error("grid dimensions must be positive"); return SG_EINVAL; }
  if (7 * nx * ny * nz >= (int64_t)INT32_MAX) { set_error("grid too large for int32 indices"); return SG_EINVAL; }
  k_poisson3d<<<grid_for(nx * ny * nz + 1), 256, 0, as_stream(stream)>>>(nx, ny, nz, offs, cols, vals);
  SG_LAUNCH_CHECK("k_poisson3d");
  return SG_OK;
}

extern "C" int sg_graph_features_block(int64_t n_block, int64_t grow0, int64_t n_global, const int32_t* offs,
                                       const int32_t* cols, const double* vals, const double* norm, int family,
                                       int64_t nx, int64_t ny, const double* coeff, double coeff_mean,
                                       double* node_out, double* edge_out, void* stream) {
  if (family == 1 && nx * ny != n_global) { set_error("meta grid does not match matrix size"); return SG_EINVAL; }
  if (grow0 < 0 || grow0 + n_block > n_global) { set_error("row block outside the matrix"); return SG_EINVAL; }
  if (n_block <= 0) return SG_OK;
  k_graph_features<<<grid_for(n_block), 256, 0, as_stream(stream)>>>(n_block, 0, grow0, n_global, offs, cols, vals,
                                                                     norm, family, nx, ny, coeff, coeff_mean,
                                                                     node_out, edge_out);
  SG_LAUNCH_CHECK("k_graph_features (block)");
  return SG_OK;
}

extern "C" int sg_norm_acc_size(void) { return NLIMB + 2; }

extern "C" int sg_norm_accum(const double* vals, int64_t nnz, int kind, uint64_t* acc_out, void* ws,
                             size_t* ws_bytes, void* stream) {
  Carve c(ws);
  unsigned long long* limbs = c.take<unsigned long long>(NLIMB);
  unsigned int* flags = c.take<unsigned int>(1);
  int64_t* seg = c.take<int64_t>(2);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (kind < 0 || kind > 2) { set_error("unknown norm kind"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  SG_CUDA(cudaMemsetAsync(limbs, 0, NLIMB * sizeof(unsigned long long), s));
  SG_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int), s));
  const int64_t h[2] = {0, nnz > 0 ? nnz : 0};
  SG_CUDA(cudaMemcpyAsync(seg, h, sizeof(h), cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    int bx = (int)ceil_div(nnz, 256);
    if (bx > 148 * 16) bx = 148 * 16;
    k_exact_accum<<<dim3(bx, 1), 256, 0, s>>>(vals, seg, kind == 1 ? 1 : 0, limbs, flags);
    SG_LAUNCH_CHECK("k_exact_accum");
  }
  k_norm_export<<<1, 32, 0, s>>>(limbs, flags, reinterpret_cast<unsigned long long*>(acc_out));
  SG_LAUNCH_CHECK("k_norm_export");
  return SG_OK;
}

extern "C" int sg_norm_from_acc(const uint64_t* acc, int64_t count, int kind, double* norm_out,
                                void* stream) {
  if (kind < 0 || kind > 2) { set_error("unknown norm kind"); return SG_EINVAL; }
  if (kind == 0 && count <= 0) { set_error("norm of a matrix with no stored entries"); return SG_EINVAL; }
  k_norm_import<<<1, 32, 0, as_stream(stream)>>>(reinterpret_cast<const unsigned long long*>(acc), count, kind,
                                                 norm_out);
  SG_LAUNCH_CHECK("k_norm_import");
  return SG_OK;
}
