// Sparsity-pattern layer: COO->CSR, validation, transpose,
// symmetry, row expansion.  Integer work, bit-exact with the reference (sparse.py).
//
// Sorting uses CUB's radix sort (header library shipped with the CUDA toolkit) keyed on the
// 64-bit (major, minor) pair — a stable sort, so the result equals np.lexsort exactly.  For the
// symmetric patterns every graph in this library has (graphfeat.py:77-78), the transpose needs
// no sort at all: sg_csr_transpose detects symmetry and computes the permutation with one
// binary search per entry (the "partner" of (i,j) is the position of (j,i)).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace sg {

__global__ void k_narrow(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t n,
                         int64_t lo, int64_t hi, int64_t shift, unsigned long long* bad) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = in[k];
    if (v < lo || v >= hi) atomicMin(bad, (unsigned long long)k);
    out[k] = (int32_t)(v + shift);
  }
}

// Segmented narrowing for block-diagonal batches: element k of segment s (seg[s] <= k <
// seg[s+1]) must satisfy 0 <= v < bound[s]; out[k] = v + shift[s].
__global__ void k_narrow_seg(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t n,
                             const int64_t* __restrict__ seg, const int64_t* __restrict__ bound,
                             const int64_t* __restrict__ shift, int n_seg, unsigned long long* bad) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_seg;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (seg[mid] <= k) lo = mid; else hi = mid;
    }
    const int64_t v = in[k];
    if (v < 0 || v >= bound[lo]) atomicMin(bad, (unsigned long long)k);
    out[k] = (int32_t)(v + shift[lo]);
  }
}

__global__ void k_coo_keys(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols,
                           int64_t nnz, int64_t n_rows, int64_t n_cols, uint64_t* keys,
                           int32_t* idx, unsigned long long* bad) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = rows[k], c = cols[k];
    unsigned long long code = 0;
    if (r < 0 || r >= n_rows) code = 1;        // "row index out of range"
    else if (c < 0 || c >= n_cols) code = 2;   // "column index out of range"
    if (code) atomicOr(bad, code);
    keys[k] = (uint64_t)(r < 0 ? 0 : r) * (uint64_t)n_cols + (uint64_t)(c < 0 ? 0 : c);
    idx[k] = (int32_t)k;
  }
}

// offs[r] = first sorted position whose major index is >= r (every r written exactly once).
__global__ void k_offsets_from_sorted(const uint64_t* __restrict__ keys, int64_t nnz,
                                      int64_t n_major, uint64_t minor_dim, int32_t* offs) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t prev = k > 0 ? (int64_t)(keys[k - 1] / minor_dim) : -1;
    int64_t cur = k < nnz ? (int64_t)(keys[k] / minor_dim) : n_major;
    for (int64_t r = prev + 1; r <= cur; ++r) offs[r] = (int32_t)k;
  }
}

__global__ void k_coo_finish(const uint64_t* __restrict__ keys, const int32_t* __restrict__ idx,
                             const double* __restrict__ vals, int64_t nnz, uint64_t n_cols,
                             int32_t* cols_out, double* vals_out, unsigned long long* first_dup) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = keys[k];
    cols_out[k] = (int32_t)(key % n_cols);
    vals_out[k] = vals[idx[k]];
    if (k + 1 < nnz && keys[k + 1] == key) atomicMin(first_dup, (unsigned long long)k);
  }
}

// Validation bits, reported in the reference's check order (sparse.py:28-43).
enum { V_OFF0 = 1, V_LAST = 2, V_MONO = 4, V_RANGE = 8, V_ORDER = 16 };

__global__ void k_validate(int64_t n_rows, int64_t n_cols, int64_t nnz,
                           const int32_t* __restrict__ offs, const int32_t* __restrict__ cols,
                           unsigned int* bits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned int b = 0;
    int64_t lo = offs[i], hi = offs[i + 1];
    if (i == 0 && lo != 0) b |= V_OFF0;
    if (i == n_rows - 1 && hi != nnz) b |= V_LAST;
    if (hi < lo) b |= V_MONO;
    if (lo >= 0 && hi <= nnz && lo <= hi) {
      for (int64_t k = lo; k < hi; ++k) {
        int32_t c = cols[k];
        if (c < 0 || c >= n_cols) b |= V_RANGE;
        if (k > lo && c <= cols[k - 1]) b |= V_ORDER;
      }
    }
    if (b) atomicOr(bits, b);
  }
}

__global__ void k_row_expand(int64_t n_rows, const int32_t* __restrict__ offs, int32_t* rows) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int32_t k = offs[i]; k < offs[i + 1]; ++k) rows[k] = (int32_t)i;
}

static inline int grid_for(int64_t n, int threads = 256) {
  int64_t g = ceil_div(n > 0 ? n : 1, threads);
  return (int)(g > 148 * 32 ? 148 * 32 : g);
}

// For entry k = (i, j): position of (j, i) by binary search in row j, or -1 if absent.
// LPR lanes share a row and search its entries in parallel (4 for stencil rows, a warp for the
// ~420-entry rows of an A^2 pattern), so a long row is not one thread's chain of dependent
// searches.
template <int LPR>
__global__ void k_partner(int64_t n, const int32_t* __restrict__ offs,
                          const int32_t* __restrict__ cols, int32_t* partner,
                          unsigned int* missing) {
  const int sub = threadIdx.x % LPR;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / LPR);
  bool miss = false;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR; i < n; i += stride) {
    const int32_t e1 = offs[i + 1];
    for (int32_t k = offs[i] + sub; k < e1; k += LPR) {
      const int32_t j = cols[k];
      int32_t lo = offs[j], hi = offs[j + 1];
      const int32_t end = hi;
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (cols[mid] < (int32_t)i) lo = mid + 1; else hi = mid;
      }
      const bool found = lo < end && cols[lo] == (int32_t)i;
      partner[k] = found ? lo : -1;
      miss |= !found;
    }
  }
  if (miss) atomicOr(missing, 1u);
}

int launch_partner(int64_t n, int64_t nnz, const int32_t* offs, const int32_t* cols, int32_t* partner,
                   unsigned int* missing, cudaStream_t s) {
  if (nnz >= 16 * n) k_partner<32><<<grid_for(32 * n), 256, 0, s>>>(n, offs, cols, partner, missing);
  else k_partner<4><<<grid_for(4 * n), 256, 0, s>>>(n, offs, cols, partner, missing);
  SG_LAUNCH_CHECK("k_partner");
  return SG_OK;
}

__global__ void k_transpose_keys(int64_t n_rows, int64_t n_cols, const int32_t* __restrict__ offs,
                                 const int32_t* __restrict__ cols, uint64_t* keys, int32_t* idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int32_t k = offs[i]; k < offs[i + 1]; ++k) {
      keys[k] = (uint64_t)cols[k] * (uint64_t)n_rows + (uint64_t)i;
      idx[k] = k;
    }
}

__global__ void k_transpose_finish(const uint64_t* __restrict__ keys, int64_t nnz, uint64_t n_rows,
                                   int32_t* cols_t) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x)
    cols_t[k] = (int32_t)(keys[k] % n_rows);
}

__global__ void k_gather(const double* __restrict__ in, const int32_t* __restrict__ perm,
                         double* __restrict__ out, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = in[perm[k]];
}

__global__ void k_copy_i32(const int32_t* __restrict__ in, int32_t* __restrict__ out, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = in[k];
}

__global__ void k_diagonal(int64_t n, const int32_t* __restrict__ offs,
                           const int32_t* __restrict__ cols, const double* __restrict__ vals,
                           double* diag, int32_t* present) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    int32_t p = 0;
    for (int32_t k = offs[i]; k < offs[i + 1]; ++k)
      if (cols[k] == (int32_t)i) { d = vals[k]; p = 1; }
    diag[i] = d;
    if (present) present[i] = p;
  }
}

// ------------------------------------------------------------------ A^2 pattern
// pattern(|A| |A|): row i = sorted union over k in cols(A_i) of cols(A_k).  One warp per row:
// gather the candidates into a per-warp shared buffer, bitonic-sort (warp-synchronous), then
// count (pass 1) or emit (pass 2) the distinct values.  Rows with more than SQ_CAP candidates
// are reported (SG_EUNSUPPORTED).
constexpr int SQ_CAP = 2048;
constexpr int SQ_WARPS = 4;

// Candidates of row i of X·Y (X rows give the k, Y rows the columns), plus i itself when
// `diag` (the Gram matrix P·Pᵀ + εI always stores its diagonal), sorted in buf[0..m).
__device__ int sq_gather_sort(int64_t i, const int32_t* __restrict__ offs, const int32_t* __restrict__ cols,
                              int32_t* buf, unsigned int* overflow, const int32_t* __restrict__ yoffs = nullptr,
                              const int32_t* __restrict__ ycols = nullptr, bool diag = false) {
  const int lane = threadIdx.x & 31;
  if (!yoffs) { yoffs = offs; ycols = cols; }
  int m = 0;
  if (diag) {
    if (lane == 0) buf[0] = (int32_t)i;
    m = 1;
  }
  for (int32_t a = offs[i]; a < offs[i + 1]; ++a) {
    const int32_t k = cols[a];
    const int32_t lo = yoffs[k], len = yoffs[k + 1] - lo;
    if (m + len > SQ_CAP) { if (lane == 0) atomicOr(overflow, 1u); return -1; }
    for (int t = lane; t < len; t += 32) buf[m + t] = ycols[lo + t];
    m += len;
  }
  int p2 = 1;
  while (p2 < m) p2 <<= 1;
  for (int t = m + lane; t < p2; t += 32) buf[t] = INT_MAX;
  __syncwarp();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = lane; t < (p2 >> 1); t += 32) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const int32_t x = buf[lo], y = buf[hi];
        if ((x > y) == up) { buf[lo] = y; buf[hi] = x; }
      }
      __syncwarp();
    }
  }
  return m;
}

__global__ void __launch_bounds__(32 * SQ_WARPS) k_square_pattern(int64_t n, const int32_t* __restrict__ offs,
                                                                 const int32_t* __restrict__ cols, int32_t* counts,
                                                                 const int32_t* __restrict__ out_offs,
                                                                 int32_t* out_cols, unsigned int* overflow) {
  __shared__ int32_t sbuf[SQ_WARPS][SQ_CAP];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* buf = sbuf[w];
  for (int64_t i = (int64_t)blockIdx.x * SQ_WARPS + w; i < n; i += (int64_t)gridDim.x * SQ_WARPS) {
    const int m = sq_gather_sort(i, offs, cols, buf, overflow);
    if (m < 0) continue;
    int written = 0;
    for (int base = 0; base < m; base += 32) {
      const int t = base + lane;
      const bool first = t < m && (t == 0 || buf[t] != buf[t - 1]);
      const unsigned int bal = __ballot_sync(0xffffffffu, first);
      if (out_cols && first) out_cols[out_offs[i] + written + __popc(bal & ((1u << lane) - 1))] = buf[t];
      written += __popc(bal);
    }
    if (!out_cols && lane == 0) counts[i] = written;
    __syncwarp();
  }
}

// Gram pattern of P·Pᵀ + εI (datasets.py:148-193, gen_synthetic): row i = {i} ∪ rows of Pᵀ over
// the columns of P's row i.  Same warp gather / bitonic sort / distinct count as above.
__global__ void __launch_bounds__(32 * SQ_WARPS) k_gram_pattern(int64_t n, const int32_t* __restrict__ p_offs,
                                                               const int32_t* __restrict__ p_cols,
                                                               const int32_t* __restrict__ pt_offs,
                                                               const int32_t* __restrict__ pt_cols, int32_t* counts,
                                                               const int32_t* __restrict__ out_offs,
                                                               int32_t* out_cols, unsigned int* overflow) {
  __shared__ int32_t sbuf[SQ_WARPS][SQ_CAP];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* buf = sbuf[w];
  for (int64_t i = (int64_t)blockIdx.x * SQ_WARPS + w; i < n; i += (int64_t)gridDim.x * SQ_WARPS) {
    const int m = sq_gather_sort(i, p_offs, p_cols, buf, overflow, pt_offs, pt_cols, true);
    if (m < 0) continue;
    int written = 0;
    for (int base = 0; base < m; base += 32) {
      const int t = base + lane;
      const bool first = t < m && (t == 0 || buf[t] != buf[t - 1]);
      const unsigned int bal = __ballot_sync(0xffffffffu, first);
      if (out_cols && first) out_cols[out_offs[i] + written + __popc(bal & ((1u << lane) - 1))] = buf[t];
      written += __popc(bal);
    }
    if (!out_cols && lane == 0) counts[i] = written;
    __syncwarp();
  }
}

// Gram values: A_ij = (sum over the columns c shared by P's rows i and j, ASCENDING c, of
// P_ic·P_jc, added one at a time to 0.0) (+ eps when i == j) -- the reference's dictionary
// accumulation visits P's column groups in ascending column order (lexsort by column, then
// row), adds acc.get(key, 0.0) + v_p·v_q, and shifts the diagonal last.  A sequential merge of
// the two sorted rows reproduces every rounding.  One warp per row, one lane per entry.
__global__ void k_gram_values(int64_t n, const int32_t* __restrict__ p_offs, const int32_t* __restrict__ p_cols,
                              const double* __restrict__ p_vals, const int32_t* __restrict__ a_offs,
                              const int32_t* __restrict__ a_cols, double shift, double* __restrict__ a_vals) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const int32_t ib = p_offs[i], ie = p_offs[i + 1];
    for (int32_t e = a_offs[i] + lane; e < a_offs[i + 1]; e += 32) {
      const int32_t j = a_cols[e];
      int32_t a = ib, b = p_offs[j];
      const int32_t be = p_offs[j + 1];
      double acc = 0.0;
      while (a < ie && b < be) {
        const int32_t ca = p_cols[a], cb = p_cols[b];
        if (ca == cb) {
          acc = __dadd_rn(acc, __dmul_rn(p_vals[a], p_vals[b]));
          ++a; ++b;
        } else if (ca < cb) {
          ++a;
        } else {
          ++b;
        }
      }
      if (j == (int32_t)i) acc = __dadd_rn(acc, shift);
      a_vals[e] = acc;
    }
  }
}

// Scatter A's values onto a superset pattern P (both CSR, sorted rows): explicit zeros elsewhere.
__global__ void k_pad_to_pattern(int64_t n, const int32_t* __restrict__ a_offs, const int32_t* __restrict__ a_cols,
                                 const double* __restrict__ a_vals, const int32_t* __restrict__ p_offs,
                                 const int32_t* __restrict__ p_cols, double* out, unsigned int* missing) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t ka = a_offs[i];
    const int32_t ea = a_offs[i + 1];
    for (int32_t kp = p_offs[i]; kp < p_offs[i + 1]; ++kp) {
      const int32_t c = p_cols[kp];
      double v = 0.0;
      if (ka < ea && a_cols[ka] == c) { v = a_vals[ka]; ++ka; }
      out[kp] = v;
    }
    if (ka != ea) atomicOr(missing, 1u);
  }
}

// Exclusive scan of counts into offsets (one block; the pattern build is not on the hot loop).
__global__ void k_scan_counts(const int32_t* __restrict__ counts, int64_t n, int32_t* offs, unsigned int* big) {
  __shared__ long long part[1024];
  const int T = blockDim.x;
  const int64_t chunk = (n + T - 1) / T;
  const int64_t lo = threadIdx.x * chunk, hi = min(n, lo + chunk);
  long long s = 0;
  for (int64_t i = lo; i < hi; ++i) s += counts[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int t = 0; t < T; ++t) { const long long v = part[t]; part[t] = acc; acc += v; }
    if (acc >= INT32_MAX) *big = 1u;
    offs[n] = (int32_t)acc;
  }
  __syncthreads();
  long long acc = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) { offs[i] = (int32_t)acc; acc += counts[i]; }
}

// Row block of a CSR matrix: rows [r0, r1), entries with r0c <= col < r1c kept (shifted by
// -r0c + col_base), in storage order.  counts[i] = kept entries of block row i.
__global__ void k_block_count(const int32_t* __restrict__ offs, const int32_t* __restrict__ cols, int64_t r0,
                              int64_t nr, int64_t c0, int64_t c1, int32_t* counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = 0;
    for (int32_t k = offs[r0 + i]; k < offs[r0 + i + 1]; ++k) c += (cols[k] >= c0 && cols[k] < c1) ? 1 : 0;
    counts[i] = c;
  }
}

__global__ void k_block_fill(const int32_t* __restrict__ offs, const int32_t* __restrict__ cols, int64_t r0,
                             int64_t nr, int64_t c0, int64_t c1, int64_t col_base, int64_t entry_base,
                             const int32_t* __restrict__ local_offs, int32_t* out_offs, int32_t* out_cols,
                             int32_t* out_src) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nr; i += (int64_t)gridDim.x * blockDim.x) {
    out_offs[i] = (int32_t)(entry_base + local_offs[i]);
    if (i == nr) continue;
    int32_t o = local_offs[i];
    for (int32_t k = offs[r0 + i]; k < offs[r0 + i + 1]; ++k) {
      const int32_t c = cols[k];
      if (c < c0 || c >= c1) continue;
      if (out_cols) out_cols[o] = (int32_t)(c - c0 + col_base);
      if (out_src) out_src[o] = k;
      ++o;
    }
  }
}

static int bits_for(uint64_t maxkey) {
  int b = 1;
  while (b < 64 && (maxkey >> b) != 0) ++b;
  return b;
}

}  // namespace sg

using namespace sg;

extern "C" int sg_narrow_index(const int64_t* in, int32_t* out, int64_t n, int64_t lo, int64_t hi,
                               int64_t shift, void* ws, size_t* ws_bytes, void* stream) {
  Carve c(ws);
  unsigned long long* bad = c.take<unsigned long long>(1);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  if (n == 0) return SG_OK;
  SG_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
  k_narrow<<<grid_for(n), 256, 0, s>>>(in, out, n, lo, hi, shift, bad);
  SG_LAUNCH_CHECK("k_narrow");
  unsigned long long h = 0;
  SG_CUDA(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  if (h != ~0ull) {
    set_error("index out of range at position %llu", h);
    return SG_EINVAL;
  }
  return SG_OK;
}

extern "C" int sg_pattern_square(int64_t n, const int32_t* offs, const int32_t* cols, int32_t* out_offs,
                                 int32_t* out_cols, int64_t* out_nnz_host, void* ws, size_t* ws_bytes, void* stream) {
  Carve c(ws);
  int32_t* counts = c.take<int32_t>(n + 1);
  unsigned int* flags = c.take<unsigned int>(2);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  const int grid = (int)(ceil_div(n > 0 ? n : 1, SQ_WARPS) < 148 * 16 ? ceil_div(n > 0 ? n : 1, SQ_WARPS) : 148 * 16);
  if (!out_cols) {  // pass 1: offsets + nnz
    SG_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned int), s));
    if (n > 0) k_square_pattern<<<grid, 32 * SQ_WARPS, 0, s>>>(n, offs, cols, counts, nullptr, nullptr, flags);
    k_scan_counts<<<1, 1024, 0, s>>>(counts, n, out_offs, flags + 1);
    SG_LAUNCH_CHECK("k_square_pattern (count)");
    unsigned int hf[2];
    int32_t nnz = 0;
    SG_CUDA(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaMemcpyAsync(&nnz, out_offs + n, sizeof(nnz), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    if (hf[0]) { set_error("a row of A^2 has more than %d candidate entries", SQ_CAP); return SG_EUNSUPPORTED; }
    if (hf[1]) { set_error("A^2 pattern exceeds the int32 index range"); return SG_EUNSUPPORTED; }
    *out_nnz_host = nnz;
    return SG_OK;
  }
  if (n > 0) k_square_pattern<<<grid, 32 * SQ_WARPS, 0, s>>>(n, offs, cols, nullptr, out_offs, out_cols, flags);
  SG_LAUNCH_CHECK("k_square_pattern (fill)");
  return SG_OK;
}

extern "C" int sg_gram_pattern(int64_t n, const int32_t* p_offs, const int32_t* p_cols, const int32_t* pt_offs,
                               const int32_t* pt_cols, int32_t* out_offs, int32_t* out_cols, int64_t* out_nnz_host,
                               void* ws, size_t* ws_bytes, void* stream) {
  Carve c(ws);
  int32_t* counts = c.take<int32_t>(n + 1);
  unsigned int* flags = c.take<unsigned int>(2);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  if (n < 1) { set_error("matrix size must be positive"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  const int grid = (int)(ceil_div(n, SQ_WARPS) < 148 * 16 ? ceil_div(n, SQ_WARPS) : 148 * 16);
  if (!out_cols) {  // pass 1: offsets + nnz
    SG_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned int), s));
    k_gram_pattern<<<grid, 32 * SQ_WARPS, 0, s>>>(n, p_offs, p_cols, pt_offs, pt_cols, counts, nullptr, nullptr, flags);
    k_scan_counts<<<1, 1024, 0, s>>>(counts, n, out_offs, flags + 1);
    SG_LAUNCH_CHECK("k_gram_pattern (count)");
    unsigned int hf[2];
    int32_t nnz = 0;
    SG_CUDA(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaMemcpyAsync(&nnz, out_offs + n, sizeof(nnz), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    if (hf[0]) { set_error("a row of P P^T has more than %d candidate entries", SQ_CAP - 1); return SG_EUNSUPPORTED; }
    if (hf[1]) { set_error("P P^T pattern exceeds the int32 index range"); return SG_EUNSUPPORTED; }
    *out_nnz_host = nnz;
    return SG_OK;
  }
  k_gram_pattern<<<grid, 32 * SQ_WARPS, 0, s>>>(n, p_offs, p_cols, pt_offs, pt_cols, nullptr, out_offs, out_cols, flags);
  SG_LAUNCH_CHECK("k_gram_pattern (fill)");
  return SG_OK;
}

extern "C" int sg_gram_values(int64_t n, const int32_t* p_offs, const int32_t* p_cols, const double* p_vals,
                              const int32_t* a_offs, const int32_t* a_cols, double shift, double* a_vals,
                              void* stream) {
  if (n < 1) { set_error("matrix size must be positive"); return SG_EINVAL; }
  const int warps_per_block = 8;
  const int64_t blocks = ceil_div(n, warps_per_block);
  k_gram_values<<<(int)(blocks < 148 * 16 ? blocks : 148 * 16), 32 * warps_per_block, 0, as_stream(stream)>>>(
      n, p_offs, p_cols, p_vals, a_offs, a_cols, shift, a_vals);
  SG_LAUNCH_CHECK("k_gram_values");
  return SG_OK;
}

extern "C" int sg_csr_pad_to_pattern(int64_t n, const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                                     const int32_t* p_offs, const int32_t* p_cols, double* out_vals, void* ws,
                                     size_t* ws_bytes, void* stream) {
  Carve c(ws);
  unsigned int* missing = c.take<unsigned int>(1);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  cudaStream_t s = as_stream(stream);
  SG_CUDA(cudaMemsetAsync(missing, 0, sizeof(unsigned int), s));
  if (n > 0) k_pad_to_pattern<<<grid_for(n), 256, 0, s>>>(n, a_offs, a_cols, a_vals, p_offs, p_cols, out_vals, missing);
  SG_LAUNCH_CHECK("k_pad_to_pattern");
  unsigned int h = 0;
  SG_CUDA(cudaMemcpyAsync(&h, missing, sizeof(h), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  if (h) { set_error("target pattern does not contain the matrix pattern"); return SG_EINVAL; }
  return SG_OK;
}

extern "C" int sg_narrow_index_segments(const int64_t* in, int32_t* out, int64_t n, const int64_t* seg_start,
                                        const int64_t* bound, const int64_t* shift, int32_t n_seg, void* ws,
                                        size_t* ws_bytes, void* stream) {
  Carve c(ws);
  unsigned long long* bad = c.take<unsigned long long>(1);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  if (n <= 0 || n_seg <= 0) return SG_OK;
  cudaStream_t s = as_stream(stream);
  SG_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
  k_narrow_seg<<<grid_for(n), 256, 0, s>>>(in, out, n, seg_start, bound, shift, n_seg, bad);
  SG_LAUNCH_CHECK("k_narrow_seg");
  unsigned long long h = 0;
  SG_CUDA(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  if (h != ~0ull) {
    set_error("index out of range at position %llu of the batch", h);
    return SG_EINVAL;
  }
  return SG_OK;
}

extern "C" int sg_csr_from_coo(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rows,
                               const int64_t* cols, const double* vals, int32_t* offs_out,
                               int32_t* cols_out, double* vals_out, int64_t* dup_host, void* ws,
                               size_t* ws_bytes, void* stream) {
  if (n_rows < 0 || n_cols < 0 || nnz < 0 || nnz >= (int64_t)INT32_MAX || n_rows >= INT32_MAX ||
      n_cols >= INT32_MAX) {
    set_error("sizes out of the supported int32 index range");
    return SG_EINVAL;
  }
  const uint64_t maxkey = (uint64_t)(n_rows > 0 ? n_rows : 1) * (uint64_t)(n_cols > 0 ? n_cols : 1);
  const int end_bit = bits_for(maxkey);
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, (int)nnz, 0, end_bit);
  Carve c(ws);
  uint64_t* k_in = c.take<uint64_t>(nnz + 1);
  uint64_t* k_out = c.take<uint64_t>(nnz + 1);
  int32_t* i_in = c.take<int32_t>(nnz + 1);
  int32_t* i_out = c.take<int32_t>(nnz + 1);
  unsigned long long* flags = c.take<unsigned long long>(2);
  void* cub_tmp = c.take<char>(cub_bytes);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  SG_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned long long), s));
  SG_CUDA(cudaMemsetAsync(flags + 1, 0xff, sizeof(unsigned long long), s));
  if (nnz > 0) {
    k_coo_keys<<<grid_for(nnz), 256, 0, s>>>(rows, cols, nnz, n_rows, n_cols, k_in, i_in, flags);
    SG_LAUNCH_CHECK("k_coo_keys");
    unsigned long long bad = 0;
    SG_CUDA(cudaMemcpyAsync(&bad, flags, sizeof(bad), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    if (bad & 1) { set_error("row index out of range"); return SG_EINVAL; }
    if (bad & 2) { set_error("column index out of range"); return SG_EINVAL; }
    size_t tb = cub_bytes;
    SG_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, k_in, k_out, i_in, i_out, (int)nnz, 0,
                                            end_bit, s));
    k_coo_finish<<<grid_for(nnz), 256, 0, s>>>(k_out, i_out, vals, nnz, (uint64_t)n_cols,
                                               cols_out, vals_out, flags + 1);
    SG_LAUNCH_CHECK("k_coo_finish");
    unsigned long long dup = 0;
    SG_CUDA(cudaMemcpyAsync(&dup, flags + 1, sizeof(dup), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    if (dup != ~0ull) {
      uint64_t key = 0;
      SG_CUDA(cudaMemcpy(&key, k_out + dup, sizeof(key), cudaMemcpyDeviceToHost));
      dup_host[0] = (int64_t)(key / (uint64_t)n_cols);
      dup_host[1] = (int64_t)(key % (uint64_t)n_cols);
      set_error("duplicate entry at (%lld, %lld)", (long long)dup_host[0], (long long)dup_host[1]);
      return SG_EDUPLICATE;
    }
  }
  k_offsets_from_sorted<<<grid_for(nnz + 1), 256, 0, s>>>(k_out, nnz, n_rows,
                                                          (uint64_t)(n_cols > 0 ? n_cols : 1),
                                                          offs_out);
  SG_LAUNCH_CHECK("k_offsets_from_sorted");
  SG_CUDA(cudaStreamSynchronize(s));
  return SG_OK;
}

extern "C" int sg_csr_validate(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* offs,
                               const int32_t* cols, void* ws, size_t* ws_bytes, void* stream) {
  Carve c(ws);
  unsigned int* bits = c.take<unsigned int>(1);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  cudaStream_t s = as_stream(stream);
  SG_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned int), s));
  unsigned int h = 0;
  if (n_rows > 0) {
    k_validate<<<grid_for(n_rows), 256, 0, s>>>(n_rows, n_cols, nnz, offs, cols, bits);
    SG_LAUNCH_CHECK("k_validate");
    SG_CUDA(cudaMemcpyAsync(&h, bits, sizeof(h), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
  } else if (nnz != 0) {
    h = V_LAST;
  }
  if (h & V_OFF0) { set_error("row_offsets[0] must be 0"); return SG_EINVAL; }
  if (h & V_LAST) { set_error("row_offsets[-1] must equal nnz"); return SG_EINVAL; }
  if (h & V_MONO) { set_error("row_offsets must be nondecreasing"); return SG_EINVAL; }
  if (h & V_RANGE) { set_error("column index out of range"); return SG_EINVAL; }
  if (h & V_ORDER) { set_error("col_indices must be strictly increasing within each row"); return SG_EINVAL; }
  return SG_OK;
}

extern "C" int sg_row_expand(int64_t n_rows, const int32_t* offs, int32_t* rows_out, void* stream) {
  if (n_rows <= 0) return SG_OK;
  k_row_expand<<<grid_for(n_rows), 256, 0, as_stream(stream)>>>(n_rows, offs, rows_out);
  SG_LAUNCH_CHECK("k_row_expand");
  return SG_OK;
}

extern "C" int sg_gather_f64(const double* in, const int32_t* perm, double* out, int64_t n,
                             void* stream) {
  if (n <= 0) return SG_OK;
  k_gather<<<grid_for(n), 256, 0, as_stream(stream)>>>(in, perm, out, n);
  SG_LAUNCH_CHECK("k_gather");
  return SG_OK;
}

extern "C" int sg_csr_diagonal(int64_t n, const int32_t* offs, const int32_t* cols,
                               const double* vals, double* diag_out, int32_t* present_out,
                               void* stream) {
  if (n <= 0) return SG_OK;
  k_diagonal<<<grid_for(n), 256, 0, as_stream(stream)>>>(n, offs, cols, vals, diag_out, present_out);
  SG_LAUNCH_CHECK("k_diagonal");
  return SG_OK;
}

extern "C" int sg_pattern_is_symmetric(int64_t n, int64_t nnz, const int32_t* offs,
                                       const int32_t* cols, int32_t* result_host, void* ws,
                                       size_t* ws_bytes, void* stream) {
  Carve c(ws);
  int32_t* partner = c.take<int32_t>(nnz + 1);
  unsigned int* missing = c.take<unsigned int>(1);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  cudaStream_t s = as_stream(stream);
  SG_CUDA(cudaMemsetAsync(missing, 0, sizeof(unsigned int), s));
  if (n > 0) {
    const int rc = launch_partner(n, nnz, offs, cols, partner, missing, s);
    if (rc) return rc;
  }
  unsigned int h = 0;
  SG_CUDA(cudaMemcpyAsync(&h, missing, sizeof(h), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  *result_host = h ? 0 : 1;
  return SG_OK;
}

extern "C" int sg_csr_transpose(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* offs,
                                const int32_t* cols, int32_t* offs_t, int32_t* cols_t,
                                int32_t* perm, void* ws, size_t* ws_bytes, void* stream) {
  const uint64_t maxkey = (uint64_t)(n_rows > 0 ? n_rows : 1) * (uint64_t)(n_cols > 0 ? n_cols : 1);
  const int end_bit = bits_for(maxkey);
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, (int)nnz, 0, end_bit);
  Carve c(ws);
  uint64_t* k_in = c.take<uint64_t>(nnz + 1);
  uint64_t* k_out = c.take<uint64_t>(nnz + 1);
  int32_t* i_in = c.take<int32_t>(nnz + 1);
  unsigned int* missing = c.take<unsigned int>(1);
  void* cub_tmp = c.take<char>(cub_bytes);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  // Fast path: square symmetric pattern => pattern(A^T) == pattern(A), perm = partner map.
  if (n_rows == n_cols && n_rows > 0) {
    SG_CUDA(cudaMemsetAsync(missing, 0, sizeof(unsigned int), s));
    const int rc = launch_partner(n_rows, nnz, offs, cols, perm, missing, s);
    if (rc) return rc;
    unsigned int h = 1;
    SG_CUDA(cudaMemcpyAsync(&h, missing, sizeof(h), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    if (!h) {
      k_copy_i32<<<grid_for(n_rows + 1), 256, 0, s>>>(offs, offs_t, n_rows + 1);
      k_copy_i32<<<grid_for(nnz), 256, 0, s>>>(cols, cols_t, nnz);
      SG_LAUNCH_CHECK("k_copy_i32");
      return SG_OK;
    }
  }
  if (nnz > 0) {
    k_transpose_keys<<<grid_for(n_rows), 256, 0, s>>>(n_rows, n_cols, offs, cols, k_in, i_in);
    SG_LAUNCH_CHECK("k_transpose_keys");
    size_t tb = cub_bytes;
    SG_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, k_in, k_out, i_in, perm, (int)nnz, 0,
                                            end_bit, s));
    k_transpose_finish<<<grid_for(nnz), 256, 0, s>>>(k_out, nnz, (uint64_t)n_rows, cols_t);
    SG_LAUNCH_CHECK("k_transpose_finish");
  }
  k_offsets_from_sorted<<<grid_for(nnz + 1), 256, 0, s>>>(k_out, nnz, n_cols,
                                                          (uint64_t)(n_rows > 0 ? n_rows : 1), offs_t);
  SG_LAUNCH_CHECK("k_offsets_from_sorted");
  return SG_OK;
}

extern "C" int sg_csr_row_block(const int32_t* offs, const int32_t* cols, int64_t r0, int64_t r1, int64_t c0,
                                int64_t c1, int64_t col_base, int64_t entry_base, int32_t* out_offs,
                                int32_t* out_cols, int32_t* out_src, int64_t* out_nnz_host, void* ws,
                                size_t* ws_bytes, void* stream) {
  const int64_t nr = r1 - r0;
  Carve c(ws);
  int32_t* counts = c.take<int32_t>(nr > 0 ? nr : 1);
  int32_t* loc = c.take<int32_t>(nr + 1);
  unsigned int* big = c.take<unsigned int>(1);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  if (nr < 0 || c1 < c0) { set_error("bad row / column range"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  SG_CUDA(cudaMemsetAsync(big, 0, sizeof(unsigned int), s));
  if (nr > 0) k_block_count<<<grid_for(nr), 256, 0, s>>>(offs, cols, r0, nr, c0, c1, counts);
  k_scan_counts<<<1, 1024, 0, s>>>(counts, nr, loc, big);
  SG_LAUNCH_CHECK("k_block_count");
  if (out_offs) {
    k_block_fill<<<grid_for(nr + 1), 256, 0, s>>>(offs, cols, r0, nr, c0, c1, col_base, entry_base, loc, out_offs,
                                                  out_cols, out_src);
    SG_LAUNCH_CHECK("k_block_fill");
  }
  if (out_nnz_host) {
    int32_t nz = 0;
    unsigned int hb = 0;
    SG_CUDA(cudaMemcpyAsync(&nz, loc + nr, sizeof(nz), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaMemcpyAsync(&hb, big, sizeof(hb), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    if (hb || entry_base + (int64_t)nz >= (int64_t)INT32_MAX) { set_error("block exceeds the int32 index range"); return SG_EINVAL; }
    *out_nnz_host = nz;
  }
  return SG_OK;
}
