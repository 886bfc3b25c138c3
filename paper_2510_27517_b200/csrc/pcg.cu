// Batched, device-resident PCG (pcg.py:131-233).
//
// A batch of independent SPD systems is stored block-diagonally (global column indices).  Rows
// are cut into TILES of PR rows that never straddle two systems; one CTA per tile.  Every dot
// product is a per-system sum of per-tile partials, reduced deterministically (fixed-shape
// trees) by the CTA that completes the system's last tile.  That CTA also runs the reference's
// scalar control flow (alpha, beta, NotSpd checks, refresh, the fresh-residual re-check,
// max_iters, the delta test, history) on device; a stopped system's tiles exit immediately in
// later launches.  The host only launches CUDA graphs of one refresh period of iterations and
// polls one counter.
//
// One iteration = three fused kernels (two more on refresh iterations):
//   K1  d' = s + beta d (on the fly for neighbours), q = A d', partial d'.q
//       [+ r_fresh = b - A x and ||r_fresh||^2 when a fresh check / certification is pending]
//   K2  x += alpha d', r' = r - alpha q (on the fly), t = G^T r', partial ||r'||^2
//   K3  s = G t + eps r' (or r' / r' * inv_diag), partial r'.s, finalizer
// Refresh iterations (i > 0, i % period == 0) replace K2 by: x += alpha d'; r' = b - A x;
// t = G^T r'.  Vector updates use the reference's roundings (no FMA), SpMVs its summation order,
// so the only arithmetic difference from numpy is the order of the dot-product reductions
// (numpy uses OpenBLAS ddot).
//
// Two storage formats for the matrices, chosen per handle:
//   DIA  (stencil patterns: <= 8 distinct diagonals, symmetric, G on A's pattern — the 2-D/3-D
//        Poisson / diffusion configs).  Values diagonal-major [ndiag][n] with a per-row presence
//        mask; no index traffic at all, every load coalesced.  G^T is never stored: row i of G^T
//        on diagonal d is G's mirror diagonal at row i + off[d].  Rows are reduced over the
//        PRESENT diagonals only, in ascending column order, so sums match CSR bit for bit.
//   CSR  (anything else): CSR-stream tiles staged through shared memory (spmv.cuh).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "spmv.cuh"
#include "tma.cuh"

namespace sg {

constexpr int PR = 256;    // rows per tile (= threads per CTA)
constexpr int PCAP = 2048; // staged nonzeros per tile (8 per row on average)
constexpr int MAXD = 8;    // DIA: max diagonals
constexpr int kMaxStageHalo = 512;  // DIA halo staging: shared memory <= 48 KB per CTA
constexpr int kSwC = PR;              // sliding window: rows per chunk
constexpr int kRpt = 4;    // DIA: rows per thread (tile = PR * kRpt rows; amortises the
                           // per-tile reduction and keeps more independent loads in flight)

enum { ST_RUN = 0, ST_CERTIFY = 1, ST_DONE = 2 };
// FL_XPEND: x still lacks alpha d' of the last fused K2+K3 (deferred x update, d' in d0 if
// FL_DPAR else d1); FL_XINT: the updated x lives in t (a fresh-residual K1 could not update x in
// place while other CTAs read it).
enum { FL_FRESH = 1, FL_XPEND = 2, FL_XINT = 4, FL_DPAR = 8 };

struct SysState {
  double norm_b, delta, delta0, dq, alpha, beta, rr, rtol2d0;
  long long i, max_iters, hist_len, fail_iter;
  double fail_value;
  int status, flags, converged, fail_kind, notspd;
  int pad[3];
};

struct Ctl {
  double rtol, eps;
  double* hist;        // [S][hcap]
  long long hcap;
  int track, delta_mode;
  unsigned int n_active;
  unsigned int snap;   // n_active seen right before the profiled iteration of a chunk
  unsigned long long apply_ns;  // one-CTA / cluster solver: device time of the applies (%globaltimer)
};

struct Dia {
  int nd;
  int halo;            // max |off|
  int W;               // 5-point grid line width (offsets {-W,-1,0,1,W}), else 0
  int off[MAXD];       // ascending column offsets
  int mir[MAXD];       // mirror diagonal: off[mir[d]] == -off[d]
  long long n;
  long long ld;        // diagonal stride: n + 2*guard (guard = max |off| zero rows on both sides,
                       // so neighbour reads never need clamping)
  const double* a;     // [nd][ld], pointer at row 0 of diagonal 0
  const double* g;     // [nd][ld]
  const double* av[MAXD];  // row-0 pointer of every diagonal of A / G
  const double* gv[MAXD];
  const unsigned char* mask;  // [n], bit d: entry (i, i+off[d]) stored
};

// SELL-32 (sliced ELLPACK, slices of 32 rows stored column-major, padded to the slice's longest
// row): entry k of row r at sbase[r/32] + 32 k + r%32, so one warp reading entry k of its 32
// rows is one coalesced transaction.  Used for CSR matrices with long rows (C4) for A and G^T,
// whose rows are summed strictly in order; row r's entries are still read in order, so the
// reference's summation orders are unchanged.  (G's numpy-pairwise rows stay CSR: measured
// faster there.)
struct Sell {
  const long long* sbase;  // [n/32 + 1]
  const int32_t* cols;
  const double* vals;
  const int32_t* offs;     // the CSR offsets (row lengths)
};

struct Dev {
  unsigned long long* trace;  // sg_pcg_set_trace: per-CTA %globaltimer stamps of the strip kernels (or null)
  int xdefer;       // sliding-window path: x += alpha d' deferred from K2+K3 to the next K1
  int sell_on;      // CSR path reads A, G^T (bit 1: also G) from their SELL-32 copies
  Sell sa, sg, sgt;
  // Row partition of ONE system (sg_pcg_set_partition / sg_pcg_set_peers).  Every system of the
  // handle is then a PARTITION: an extended local system = owned rows [own0, own1) plus ghost
  // rows on either side (3 half-bandwidths deep).  The kernels run over the whole extended
  // system as usual; only the owned rows enter the dot products and store s, and the first /
  // last owned rows of s are also stored into the neighbour partitions' ghost rows (push_lo /
  // push_hi: the same vector of the same handle in group mode, peer-mapped NVLink memory in peer
  // mode).  Every other ghost value stays exact by redundant computation.  The
  // two-scalar reductions combine the partitions' sums in partition order (part_fin).
  int part;  // 0 = off, 1 = group (all partitions in this handle), 2 = peer (one per rank)
  const long long* own0;  // [S] owned rows (absolute; = the system's rows when part == 0)
  const long long* own1;
  const long long* plo;   // [S] rows pushed down (into partition sys-1's top ghost rows)
  const long long* phi;   // [S] rows pushed up (into partition sys+1's bottom ghost rows)
  double* const* push_lo; // [S] destination of own row own0 (nullptr: none)
  double* const* push_hi; // [S] destination of own row own1 - phi
  double* gsum;           // group: [S][2] per-partition sums; peer: [2 parity][R][2] (IPC memory)
  unsigned int* grp;      // group: arrivals of the current reduction
  int nsys;               // partitions in this handle (group mode)
  // peer mode (one partition per rank, NVLink peer memory opened with CUDA IPC)
  int rank, nranks;
  double* peer_gsum[8];         // every rank's gsum block (own = local)
  unsigned int* peer_flag[8];   // every rank's flag array [R]: slot q = last epoch rank q published
  unsigned int* epoch;          // local reduction counter (thread 0 of a reducing CTA)
  // tile table
  const long long* blk_r0;
  const int* blk_sys;
  const int* sys_blk0;
  const long long* sys_r1;
  int tile;  // rows per tile: PR (CSR) or PR * kRpt (DIA)
  // sliding-window range table (halo-staged DIA): ranges of <= rng_len rows inside one system
  long long rng_len;
  const long long* rng_r0;
  const int* rng_sys;
  const int* sys_rng0;
  // matrices (CSR)
  const int32_t *a_offs, *a_cols; const double* a_vals;
  const int32_t *g_offs, *g_cols; const double* g_vals;
  const int32_t *gt_offs, *gt_cols; const double* gt_vals;
  const double* inv_diag;
  Dia dia;
  // coefficient stencil (sg_pcg_set_stencil): A regenerated from the node coefficients of
  // gen_poisson2d inside the sliding-window K1 instead of streaming its diagonals
  const double* coef;  // [n] with the diagonals' guard rows
  double ihx2, ihy2;
  // wide-grid strips: G + mask of every (strip, line) segment as one contiguous block (see
  // k_strip_gblocks), so K2+K3 fetches a line's G with ONE bulk copy
  const unsigned char* gblk;
  long long gblk_L;  // extended lines per strip (every system's lines + 4 zero lines)
  // vectors
  double *b, *x, *r0, *r1, *d0, *d1, *q, *s, *t;
  // reduction scratch
  double* pp;               // per-CTA partials [nblk][2]
  unsigned int* counter;    // [S]
  SysState* st;
  Ctl* ctl;
};

__global__ void k_snapshot(Ctl* c) { c->snap = c->n_active; }

__global__ void k_max_row(const int32_t* __restrict__ offs, int64_t n, unsigned int* out) {
  unsigned int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned int)(offs[i + 1] - offs[i]));
  atomicMax(out, m);
}

__global__ void k_differ(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n, unsigned int* flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    if (a[k] != b[k]) { *flag = 1u; return; }
}

// ------------------------------------------------------------------ pattern fingerprint
// A handle's formats (DIA offset set, strip width, SELL column copies, tile / range tables, row
// lengths) are derived from the CSR PATTERNS at creation, while the caller may refill the same
// index buffers between solves (batch.py refills its device CSR in place).  Every solve
// fingerprints the patterns and rebuilds the handle when they moved, so a stale plan can never
// drop entries.  The fingerprint is an order-independent sum (mod 2^64) of a 64-bit mix of
// (position, value) over offs[0..n] and cols[0..offs[n]): deterministic, one read of the indices.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_pattern_hash(const int32_t* __restrict__ offs, const int32_t* __restrict__ cols, int64_t n,
                               unsigned long long salt, unsigned long long* out) {
  const int64_t nnz = offs[n];
  const int64_t tot = n + 1 + (nnz > 0 ? nnz : 0);
  unsigned long long h = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < tot; k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned int v = (unsigned int)(k <= n ? offs[k] : cols[k - n - 1]);
    h += mix64(((unsigned long long)k << 1) ^ ((unsigned long long)v << 40) ^ ((unsigned long long)v >> 24) ^ salt);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

// ------------------------------------------------------------------ DIA detection / conversion
// Insert every (col - row) into a 16-slot device set; overflow => not DIA-able.
__global__ void k_dia_offsets(const int32_t* __restrict__ offs, const int32_t* __restrict__ cols, int64_t n,
                              int* slots, int* nslots, int* overflow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int32_t k = offs[i]; k < offs[i + 1]; ++k) {
      const int o = cols[k] - (int)i;
      bool found = false;
      const int cnt = min(*(volatile int*)nslots, 16);
      for (int s = 0; s < cnt && !found; ++s) found = ((volatile int*)slots)[s] == o;
      if (found) continue;
      for (int s = 0; s < 16; ++s) {
        const int prev = atomicCAS(&slots[s], INT_MIN, o);
        if (prev == INT_MIN) { atomicMax(nslots, s + 1); found = true; break; }
        if (prev == o) { found = true; break; }
      }
      if (!found) *overflow = 1;
    }
  }
}

// CSR -> diagonal-major values (+ presence mask).  Every slot of every row is written.  An entry
// on a diagonal outside the handle's offset set sets *unmatched (the solve fails loudly instead
// of dropping it; the pattern fingerprint normally rebuilds the handle before this can happen).
__global__ void k_csr_to_dia(const int32_t* __restrict__ offs, const int32_t* __restrict__ cols,
                             const double* __restrict__ vals, int64_t n, Dia dia, double* out,
                             unsigned char* mask, unsigned int* unmatched) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v[MAXD];
#pragma unroll
    for (int d = 0; d < MAXD; ++d) v[d] = 0.0;
    unsigned int m = 0;
    for (int32_t k = offs[i]; k < offs[i + 1]; ++k) {
      const int o = cols[k] - (int)i;
      bool hit = false;
#pragma unroll
      for (int d = 0; d < MAXD; ++d)
        if (d < dia.nd && dia.off[d] == o) { v[d] = vals[k]; m |= 1u << d; hit = true; }
      if (!hit) *unmatched = 1u;
    }
#pragma unroll
    for (int d = 0; d < MAXD; ++d)
      if (d < dia.nd) out[(int64_t)d * dia.ld + i] = v[d];
    if (mask) mask[i] = (unsigned char)m;
  }
}

// CSR -> SELL-32 (values, or column indices when vals == null); padding entries stay as set.
__global__ void k_csr_to_sell(int64_t n, const int32_t* __restrict__ offs, const int32_t* __restrict__ cols,
                              const double* __restrict__ vals, const long long* __restrict__ sbase,
                              int32_t* __restrict__ scols, double* __restrict__ svals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const long long b = sbase[i >> 5] + (i & 31);
    for (int32_t k = offs[i], e = 0; k < offs[i + 1]; ++k, ++e) {
      if (svals) svals[b + 32LL * e] = vals[k];
      else scols[b + 32LL * e] = cols[k];
    }
  }
}

// ------------------------------------------------------------------ shared per-tile plumbing
__device__ __forceinline__ void block_rows(const Dev& D, int& sys, long long& r0, long long& r1) {
  sys = D.blk_sys[blockIdx.x];
  r0 = D.blk_r0[blockIdx.x];
  const long long e = r0 + D.tile;
  const long long se = D.sys_r1[sys];
  r1 = e < se ? e : se;
}

// Timeline probe (sg_pcg_set_trace, off unless a buffer is set): thread 0 of CTA b stamps slot
// `slot` (0 entry, 1 end of the stream, 2 after the arrival, 3 finaliser done) of kernel `kid`;
// slot 4 holds the SM the CTA ran on.
__device__ __forceinline__ void trace_stamp(const Dev& D, int kid, int slot) {
  if (D.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    D.trace[(size_t)kid * 16384 + 8 * blockIdx.x + slot] = t;
    if (slot == 0) {
      unsigned int smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      D.trace[(size_t)kid * 16384 + 8 * blockIdx.x + 4] = smid;
    }
  }
}

// Publish this CTA's two partials; returns true in ALL threads of the last CTA of `sys`.
// `sb0`: the per-system first-CTA table of the launch (tiles, or sliding-window ranges).
__device__ __forceinline__ bool arrive(const Dev& D, const int* sb0, int sys, double p0, double p1, double* red,
                                       int* flag) {
  if (D.part == 2) __threadfence_system();  // every thread's s-halo peer stores precede the arrival
  double a = p0, b = p1;
  block_sum2(a, b);
  if (threadIdx.x == 0) {
    D.pp[2 * blockIdx.x + 0] = a;
    D.pp[2 * blockIdx.x + 1] = b;
    __threadfence();
    const unsigned int nb = (unsigned)(sb0[sys + 1] - sb0[sys]);
    const unsigned int old = atomicAdd(&D.counter[sys], 1u);
    *flag = (old == nb - 1);
  }
  __syncthreads();
  const bool last = *flag;
  if (last) __threadfence();
  return last;
}
__device__ __forceinline__ bool arrive(const Dev& D, int sys, double p0, double p1, double* red, int* flag) {
  return arrive(D, D.sys_blk0, sys, p0, p1, red, flag);
}

// Deterministic per-system sum of partial slot `which` (valid in thread 0).
__device__ __forceinline__ double gather_partials(const Dev& D, const int* sb0, int sys, int which, double* red) {
  const int b0 = sb0[sys], b1 = sb0[sys + 1];
  double v = 0.0;
  for (int b = b0 + threadIdx.x; b < b1; b += blockDim.x) v += __ldcg(&D.pp[2 * b + which]);
  return block_sum(v, red);
}
// Both partial slots of `sys` in one pass (one round of loads, one pair of barriers); each value
// is summed exactly as gather_partials sums it.
__device__ __forceinline__ void gather_partials2(const Dev& D, const int* sb0, int sys, double& v0, double& v1) {
  const int b0 = sb0[sys], b1 = sb0[sys + 1];
  v0 = 0.0;
  v1 = 0.0;
  for (int b = b0 + threadIdx.x; b < b1; b += blockDim.x) {
    const double2 pv = __ldcg(reinterpret_cast<const double2*>(D.pp) + b);
    v0 += pv.x;
    v1 += pv.y;
  }
  block_sum2(v0, v1);
}
__device__ __forceinline__ double gather_partials(const Dev& D, int sys, int which, double* red) {
  return gather_partials(D, D.sys_blk0, sys, which, red);
}

__device__ __forceinline__ void finish(const Dev& D, SysState& S, int conv, bool pri = true) {
  S.converged = conv;
  S.status = ST_DONE;
  if (pri) atomicSub(&D.ctl->n_active, 1u);  // pri: the one copy of a replicated state that reports
}

// Owned-row window and s-push targets of one partition (whole system when not partitioned).
struct Own {
  long long o0, o1, pl, ph;
  double* dl;
  double* dh;
};
__device__ __forceinline__ Own own_of(const Dev& D, int sys) {
  Own w;
  w.o0 = D.own0[sys];
  w.o1 = D.own1[sys];
  if (D.part) {
    w.pl = D.plo[sys]; w.ph = D.phi[sys]; w.dl = D.push_lo[sys]; w.dh = D.push_hi[sys];
  } else {
    w.pl = w.ph = 0; w.dl = w.dh = nullptr;
  }
  return w;
}
__device__ __forceinline__ bool owned(const Own& w, long long i) { return i >= w.o0 && i < w.o1; }
// The streamed kernels take the partition logic as a template flag: without it the owned-row
// tests fold away and the push branch disappears (no registers spent on it: K2+K3 keeps 3 CTAs
// per SM).
template <bool PART>
__device__ __forceinline__ Own own_get(const Dev& D, int sys) {
  if constexpr (PART) return own_of(D, sys);
  else return Own{LLONG_MIN, LLONG_MAX, 0, 0, nullptr, nullptr};
}
// s of an owned row: local store plus the pushes into the neighbours' ghost rows
__device__ __forceinline__ void store_s(const Dev& D, const Own& w, long long i, double v) {
  D.s[i] = v;
  if (w.dl && i - w.o0 < w.pl) w.dl[i - w.o0] = v;
  if (w.dh && w.o1 - i <= w.ph) w.dh[i - (w.o1 - w.ph)] = v;
}

__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void put_hist(const Dev& D, int sys, long long i, double v, bool pri = true) {
  if (!pri) return;
  const Ctl& c = *D.ctl;
  if (c.track && i < c.hcap) c.hist[(long long)sys * c.hcap + i] = v;
}

// ------------------------------------------------------------------ finalizers (thread 0)
__device__ void fin_setup1(const Dev& D, int sys, double bb) {
  SysState& S = D.st[sys];
  S.norm_b = __dsqrt_rn(bb);
  S.rr = bb;
  D.counter[sys] = 0;
}

__device__ void fin_setup2(const Dev& D, int sys, double rs) {
  SysState& S = D.st[sys];
  D.counter[sys] = 0;
  const Ctl& c = *D.ctl;
  S.i = 0;
  S.beta = 0.0;
  S.flags = 0;
  S.notspd = 0;
  S.converged = 0;
  S.hist_len = 1;
  if (S.norm_b == 0.0) {  // pcg.py:159-164
    put_hist(D, sys, 0, 0.0);
    finish(D, S, 1);
    return;
  }
  put_hist(D, sys, 0, __ddiv_rn(__dsqrt_rn(S.rr), S.norm_b));
  S.delta = rs;
  if (rs < 0.0) {  // pcg.py:171-172
    S.notspd = 1; S.fail_iter = 0; S.fail_value = rs; S.fail_kind = 2;
    finish(D, S, 0);
    return;
  }
  S.delta0 = rs;
  S.rtol2d0 = mul(mul(c.rtol, c.rtol), rs);
  if (c.delta_mode) {
    if (S.max_iters <= 0 || rs <= S.rtol2d0) S.status = ST_CERTIFY;
  } else if (S.max_iters <= 0) {
    finish(D, S, 0);
  }
}

// The finalisers act on a SysState reference: the system's state in global memory (the
// multi-kernel and one-CTA paths) or a shared-memory copy (k_pcg_smem).
__device__ void fin_k1_s(const Dev& D, SysState& S, int sys, bool run, double dq, double rrf, bool pri = true) {
  D.counter[sys] = 0;
  const Ctl& c = *D.ctl;
  if (!run) {  // delta-test certification (pcg.py:217-220)
    const double rel = __ddiv_rn(__dsqrt_rn(rrf), S.norm_b);
    finish(D, S, rel <= c.rtol, pri);
    return;
  }
  if (S.flags & FL_FRESH) {  // pcg.py:208-215
    S.flags &= ~FL_FRESH;
    const double rel = __ddiv_rn(__dsqrt_rn(rrf), S.norm_b);
    put_hist(D, sys, S.i, rel, pri);
    if (rel <= c.rtol) { finish(D, S, 1, pri); return; }
    if (S.i >= S.max_iters) { finish(D, S, 0, pri); return; }
  }
  if (dq <= 0.0) {  // pcg.py:182-184
    S.notspd = 1; S.fail_iter = S.i; S.fail_value = dq; S.fail_kind = 1;
    finish(D, S, 0, pri);
    return;
  }
  S.dq = dq;
  S.alpha = __ddiv_rn(S.delta, dq);
}
__device__ void fin_k1(const Dev& D, int sys, bool run, double dq, double rrf) {
  fin_k1_s(D, D.st[sys], sys, run, dq, rrf);
}

__device__ void fin_rr(const Dev& D, int sys, double rr) {
  D.st[sys].rr = rr;
  D.counter[sys] = 0;
}

__device__ void fin_k3_s(const Dev& D, SysState& S, int sys, double rs, int refreshed, bool pri = true) {
  D.counter[sys] = 0;
  const Ctl& c = *D.ctl;
  const double delta_old = S.delta;
  S.delta = rs;
  if (rs < 0.0) {  // pcg.py:196-198
    S.notspd = 1; S.fail_iter = S.i; S.fail_value = rs; S.fail_kind = 2;
    finish(D, S, 0, pri);
    return;
  }
  S.beta = __ddiv_rn(rs, delta_old);
  S.i += 1;
  const double rel = __ddiv_rn(__dsqrt_rn(S.rr), S.norm_b);
  put_hist(D, sys, S.i, rel, pri);
  S.hist_len = S.i + 1;
  if (!c.delta_mode) {
    if (rel <= c.rtol) {
      if (refreshed) { finish(D, S, 1, pri); return; }
      S.flags |= FL_FRESH;
    } else if (S.i >= S.max_iters) {
      finish(D, S, 0, pri);
    }
  } else if (S.i >= S.max_iters || rs <= S.rtol2d0) {
    S.status = ST_CERTIFY;
  }
}
__device__ void fin_k3(const Dev& D, int sys, double rs, int refreshed) {
  fin_k3_s(D, D.st[sys], sys, rs, refreshed);
}

// ------------------------------------------------------------------ partition reductions
enum { FIN_SETUP1 = 0, FIN_SETUP2 = 1, FIN_K1 = 2, FIN_RR = 3, FIN_K3 = 4, FIN_K23 = 5 };

__device__ void run_fin(const Dev& D, int sys, int kind, double v0, double v1, int arg) {
  switch (kind) {
    case FIN_SETUP1: fin_setup1(D, sys, v0); break;
    case FIN_SETUP2: fin_setup2(D, sys, v0); break;
    case FIN_K1: fin_k1(D, sys, arg != 0, v0, v1); break;
    case FIN_RR: fin_rr(D, sys, v0); break;
    case FIN_K3: fin_k3(D, sys, v0, arg); break;
    default: D.st[sys].rr = v0; fin_k3(D, sys, v1, arg); break;
  }
}

// Thread 0 of the last CTA of partition `sys` to finish a reducing kernel, with the partition's
// sums (v0, v1).  The reference control flow then runs on the sums over ALL partitions, added
// in partition order (0.0 + p0 + p1 + ...), identically for every partition:
//  group (1): the last partition to arrive adds the published sums and finalises every
//    partition's state (all partitions run in the same launch: no waiting);
//  peer (2): the partition stores its sums into every rank's gsum (NVLink peer stores, parity
//    double-buffered by reduction epoch), releases its epoch flag on every rank, waits for all
//    ranks' flags of this epoch in local memory, and finalises its own state.  The flag also
//    orders the s-halo peer stores every CTA issued before arriving (arrive fences at system
//    scope in peer mode).
__device__ void part_fin(const Dev& D, int sys, int kind, double v0, double v1, int arg) {
  D.counter[sys] = 0;
  if (D.part == 1) {
    D.gsum[2 * sys + 0] = v0;
    D.gsum[2 * sys + 1] = v1;
    __threadfence();
    if (atomicAdd(D.grp, 1u) != (unsigned int)D.nsys - 1u) return;
    __threadfence();
    double s0 = 0.0, s1 = 0.0;
    for (int q = 0; q < D.nsys; ++q) {
      s0 = add(s0, __ldcg(&D.gsum[2 * q + 0]));
      s1 = add(s1, __ldcg(&D.gsum[2 * q + 1]));
    }
    for (int q = 0; q < D.nsys; ++q) run_fin(D, q, kind, s0, s1, arg);
    *D.grp = 0u;
    return;
  }
  const unsigned int e = *D.epoch + 1u;
  *D.epoch = e;
  const int par = (int)(e & 1u), R = D.nranks, me = D.rank;
  for (int q = 0; q < R; ++q) {
    double* g = D.peer_gsum[q] + 2 * (par * R + me);
    g[0] = v0;
    g[1] = v1;
  }
  __threadfence_system();
  for (int q = 0; q < R; ++q) st_release_sys(D.peer_flag[q] + me, e);
  const unsigned int* mine = D.peer_flag[me];
  for (int q = 0; q < R; ++q)
    while ((int)(ld_acquire_sys(mine + q) - e) < 0) {
    }
  const double* g = D.peer_gsum[me] + 2 * par * R;
  double s0 = 0.0, s1 = 0.0;
  for (int q = 0; q < R; ++q) {
    s0 = add(s0, __ldcv(&g[2 * q + 0]));
    s1 = add(s1, __ldcv(&g[2 * q + 1]));
  }
  run_fin(D, sys, kind, s0, s1, arg);
}

// ------------------------------------------------------------------ row operators
// CSR: a staged RowTile.  DIA: diagonal-major values + mask.  Both expose
//   A(i, X)  : numpy-order  sum_k A_ik X(col_k)
//   G(i, X)  : numpy-order  sum_k G_ik X(col_k)
//   Gt(i, X) : add.at order sum_k (G^T)_ik X(col_k)
template <bool SH>
struct CsrOps {
  const RowTile<PR, PCAP>* T;
  long long r0;
  const int32_t* cols;
  const double* vals;
  template <int ORDER, int XM>
  __device__ __forceinline__ double row(long long i, const XF& f) const {
    return tile_row_dot<ORDER, SH, XM>(*T, (int)(i - r0), cols, vals, f);
  }
};

// numpy-order reduction over the present diagonals of row i of a diagonal-major matrix.
// Loads are issued unconditionally first (padded slots are zeros; neighbour rows outside the
// matrix land in the zero guard bands of every vector / diagonal array, so no clamping), so no
// load waits for the mask; the mask only selects which products enter the sum, in the
// reference's order.  32-bit row indices (n < 2^31) and per-diagonal base pointers keep the
// address arithmetic to one IMAD.WIDE per load.
// Branch-free: every sum is evaluated and kept or dropped by selects, so the products of all
// diagonals are issued together and the dependent adds form one short chain.
template <int ND>
__device__ __forceinline__ double combine_numpy(const double (&p)[ND], unsigned int m) {
  if (m == (1u << ND) - 1u) {  // interior row, every diagonal present: the same adds, no selects
    double s = add(0.0, p[1 < ND ? 1 : 0]);
#pragma unroll
    for (int d = 2; d < ND; ++d) s = add(s, p[d]);
    return ND > 1 ? add(p[0], s) : p[0];
  }
  double first = 0.0, s = 0.0;
  bool have = false, more = false;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    const bool pr = (m >> d) & 1u;
    const double sn = add(s, p[d]);
    first = (pr && !have) ? p[d] : first;
    s = (pr && have) ? sn : s;
    more = more || (pr && have);
    have = have || pr;
  }
  return more ? add(first, s) : first;
}

// Sequential (add.at order) sum of the present products, branch-free.
template <int ND>
__device__ __forceinline__ double combine_seq(const double (&p)[ND], unsigned int m) {
  if (m == (1u << ND) - 1u) {  // every entry present: the same adds, no selects
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < ND; ++d) s = add(s, p[d]);
    return s;
  }
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    const double sn = add(s, p[d]);
    s = ((m >> d) & 1u) ? sn : s;
  }
  return s;
}

template <int ND, int XM>
__device__ __forceinline__ double dia_row_numpy(const Dia& dd, const double* const* Vd, int i, unsigned int m,
                                                const XF& f) {
  constexpr int NA = ND > 0 ? ND : 1;
  double a[NA], x[NA], p[NA];
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    a[d] = __ldg(Vd[d] + i);
    x[d] = xval<XM>(f, i + dd.off[d]);
  }
#pragma unroll
  for (int d = 0; d < ND; ++d) p[d] = mul(a[d], x[d]);
  return combine_numpy<NA>(p, m);
}

// Same numpy-order row reduction for an exactly SYMMETRIC matrix stored by its lower half: the
// entry on an upper diagonal d (off > 0) is read from the mirror (lower) diagonal at row
// i + off, so the upper diagonals are never streamed from HBM.
template <int ND, int XM>
__device__ __forceinline__ double dia_row_numpy_sym(const Dia& dd, const double* const* Vd, int i, unsigned int m,
                                                    const XF& f) {
  constexpr int NA = ND > 0 ? ND : 1;
  double a[NA], x[NA], p[NA];
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    const int j = i + dd.off[d];
    a[d] = dd.off[d] > 0 ? __ldg(Vd[dd.mir[d]] + j) : __ldg(Vd[d] + i);
    x[d] = xval<XM>(f, j);
  }
#pragma unroll
  for (int d = 0; d < ND; ++d) p[d] = mul(a[d], x[d]);
  return combine_numpy<NA>(p, m);
}

// Bitwise check that a diagonal-major matrix equals its transpose on the stored pattern.
__global__ void k_dia_symcheck(Dia dia, unsigned int* asym) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < dia.n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned int m = dia.mask[i];
    for (int d = 0; d < dia.nd; ++d)
      if ((m & (1u << d)) && dia.off[d] > 0) {
        const double up = dia.av[d][i];
        const double lo = dia.av[dia.mir[d]][i + dia.off[d]];
        if (__double_as_longlong(up) != __double_as_longlong(lo)) { *asym = 1u; return; }
      }
  }
}

// gen_poisson2d's entries of one row (datasets.py:110-137) from the node coefficients c0 (row),
// cs / cw / ce / cn (rows i - W, i - 1, i + 1, i + W) and the row's presence mask (bits in the
// ascending offset order {-W, -1, 0, 1, W}): faces are arithmetic means, a wall face keeps the
// node's own value (a missing neighbour = a wall), off-diagonals are -face / h^2 and the
// diagonal (w + e) / hx^2 + (s + n) / hy^2 -- numpy's roundings, no FMA, so bitwise its A.
__device__ __forceinline__ void stencil5(double c0, double cs, double cw, double ce, double cn, unsigned int m,
                                         double ihx2, double ihy2, double (&a)[5]) {
  const double fs = (m & 1u) ? mul(0.5, add(c0, cs)) : c0;
  const double fw = (m & 2u) ? mul(0.5, add(c0, cw)) : c0;
  const double fe = (m & 8u) ? mul(0.5, add(c0, ce)) : c0;
  const double fn = (m & 16u) ? mul(0.5, add(c0, cn)) : c0;
  a[0] = -mul(fs, ihy2);
  a[1] = -mul(fw, ihx2);
  a[2] = add(mul(add(fw, fe), ihx2), mul(add(fs, fn), ihy2));
  a[3] = -mul(fe, ihx2);
  a[4] = -mul(fn, ihy2);
}

// Bitwise check that the stored 5-point DIA matrix is exactly gen_poisson2d's A of `coef`
// (every stored entry of every row); any mismatch disables the coefficient stencil.
__global__ void k_stencil_check(Dia dia, const double* __restrict__ coef, double ihx2, double ihy2,
                                unsigned int* bad) {
  const int W = dia.off[4];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < dia.n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned int m = dia.mask[i];
    double a[5];
    stencil5(coef[i], coef[i - W], coef[i - 1], coef[i + 1], coef[i + W], m, ihx2, ihy2, a);
#pragma unroll
    for (int d = 0; d < 5; ++d)
      if (((m >> d) & 1u) && __double_as_longlong(a[d]) != __double_as_longlong(dia.av[d][i])) { *bad = 1u; return; }
  }
}

// add.at order over row i of G^T, read from G's mirror diagonals.
template <int ND, int XM>
__device__ __forceinline__ double dia_row_t_seq(const Dia& dd, const double* const* Vd, int i, unsigned int m,
                                                const XF& f) {
  constexpr int NA = ND > 0 ? ND : 1;
  double a[NA], x[NA];
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    const int j = i + dd.off[d];
    a[d] = __ldg(Vd[dd.mir[d]] + j);
    x[d] = xval<XM>(f, j);
  }
  double p[NA];
#pragma unroll
  for (int d = 0; d < ND; ++d) p[d] = mul(a[d], x[d]);
  return combine_seq<NA>(p, m);
}

// ------------------------------------------------------------------ kernels
// FMT 0 = CSR (SH: short rows), FMT 1 = DIA with ND diagonals.
template <int FMT, int ND>
struct Fmt {};

#define SG_KERNEL_PROLOGUE                      \
  __shared__ RowTile<PR, (FMT == 0 ? PCAP : 4)> T; \
  __shared__ double red[PR / 32];               \
  __shared__ int flag;                          \
  int sys; long long r0, r1;                    \
  block_rows(D, sys, r0, r1);                   \
  const Own ow = own_of(D, sys);                \
  constexpr int RPT = FMT >= 1 ? kRpt : 1;      \
  (void)T; (void)ow;

template <int ORDER, int XM>
__device__ __noinline__ double row_sell(const double* __restrict__ sv, const int32_t* __restrict__ sc, int len,
                                        XF f) {
  auto p = [&](int64_t k) { return mul(__ldg(sv + 32 * k), xval<XM>(f, __ldg(sc + 32 * k))); };
  if (ORDER == kOrderSeq) return sequential_sum(p, 0, len);
  return reduceat_sum(p, 0, len);
}

template <int ORDER, int XM>
__device__ __forceinline__ double sell_row(const Sell& S, long long i, const XF& f) {
  const long long b = S.sbase[i >> 5] + (i & 31);
  return row_sell<ORDER, XM>(S.vals + b, S.cols + b, S.offs[i + 1] - S.offs[i], f);
}

// A-row (numpy order) for either format.
template <int FMT, int ND, bool SH, int XM>
__device__ __forceinline__ double rowA(const Dev& D, const RowTile<PR, (FMT == 0 ? PCAP : 4)>& T, long long i,
                                       long long r0, unsigned int m, const XF& f) {
  if (FMT == 1) return dia_row_numpy<ND, XM>(D.dia, D.dia.av, (int)i, m, f);
  if (FMT == 2) return dia_row_numpy_sym<ND, XM>(D.dia, D.dia.av, (int)i, m, f);
  if (FMT == 0 && D.sell_on) return sell_row<kOrderNumpy, XM>(D.sa, i, f);
  return tile_row_dot<kOrderNumpy, SH, XM>(*reinterpret_cast<const RowTile<PR, PCAP>*>(&T), (int)(i - r0),
                                           D.a_cols, D.a_vals, f);
}
template <int FMT, int ND, bool SH, int XM>
__device__ __forceinline__ double rowG(const Dev& D, const RowTile<PR, (FMT == 0 ? PCAP : 4)>& T, long long i,
                                       long long r0, unsigned int m, const XF& f) {
  if (FMT >= 1) return dia_row_numpy<ND, XM>(D.dia, D.dia.gv, (int)i, m, f);
  if (D.sell_on & 2) return sell_row<kOrderNumpy, XM>(D.sg, i, f);
  return tile_row_dot<kOrderNumpy, SH, XM>(*reinterpret_cast<const RowTile<PR, PCAP>*>(&T), (int)(i - r0),
                                           D.g_cols, D.g_vals, f);
}
template <int FMT, int ND, bool SH, int XM>
__device__ __forceinline__ double rowGt(const Dev& D, const RowTile<PR, (FMT == 0 ? PCAP : 4)>& T, long long i,
                                        long long r0, unsigned int m, const XF& f) {
  if (FMT >= 1) return dia_row_t_seq<ND, XM>(D.dia, D.dia.gv, (int)i, m, f);
  if (D.sell_on) return sell_row<kOrderSeq, XM>(D.sgt, i, f);
  return tile_row_dot<kOrderSeq, SH, XM>(*reinterpret_cast<const RowTile<PR, PCAP>*>(&T), (int)(i - r0),
                                         D.gt_cols, D.gt_vals, f);
}

template <int FMT>
__device__ __forceinline__ void stage(const Dev& D, RowTile<PR, (FMT == 0 ? PCAP : 4)>& T, long long r0,
                                      long long r1, const int32_t* offs, const int32_t* cols, const double* vals) {
  // A and G^T rows come from their SELL copies when those exist; G (and everything else) stages
  const bool sell = D.sell_on && (vals == D.a_vals || vals == D.gt_vals);
  if (FMT == 0 && !sell) stage_rows(*reinterpret_cast<RowTile<PR, PCAP>*>(&T), r0, r1, offs, cols, vals);
}

__device__ __forceinline__ unsigned int dmask(const Dev& D, long long i, long long r1, int FMT) {
  return (FMT >= 1 && i < r1) ? (unsigned int)D.dia.mask[i] : 0u;
}

// r = b; d = 0; x = 0; t = G^T b; partial ||b||^2
template <int PRE, int FMT, int ND, bool SH>
__global__ void __launch_bounds__(PR, FMT >= 1 ? 8 : 1) k_setup1(Dev D) {
  SG_KERNEL_PROLOGUE
  if (PRE == SG_PRECOND_LEARNED) stage<FMT>(D, T, r0, r1, D.gt_offs, D.gt_cols, D.gt_vals);
  double pbb = 0.0;
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const long long i = r0 + (long long)rr * PR + threadIdx.x;
    if (i >= r1) continue;
    const unsigned int m = dmask(D, i, r1, FMT);
    const double bi = D.b[i];
    D.r0[i] = bi;
    D.d0[i] = 0.0;
    D.d1[i] = 0.0;
    D.x[i] = 0.0;
    if (owned(ow, i)) pbb += mul(bi, bi);
    if (PRE == SG_PRECOND_LEARNED) D.t[i] = rowGt<FMT, ND, SH, 0>(D, T, i, r0, m, XF{D.b, nullptr, 0.0});
  }
  if (arrive(D, sys, pbb, 0.0, red, &flag)) {
    const double bb = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) { if (D.part) part_fin(D, sys, FIN_SETUP1, bb, 0.0, 0); else fin_setup1(D, sys, bb); }
  }
}

template <int PRE, int FMT, int ND, bool SH>
__device__ __forceinline__ double apply_row(const Dev& D, const RowTile<PR, (FMT == 0 ? PCAP : 4)>& T,
                                            long long i, long long r0, unsigned int m, const double* r,
                                            double eps) {
  if (PRE == SG_PRECOND_IDENTITY) return r[i];
  if (PRE == SG_PRECOND_JACOBI) return mul(r[i], D.inv_diag[i]);
  const double y = rowG<FMT, ND, SH, 0>(D, T, i, r0, m, XF{D.t, nullptr, 0.0});
  return add(y, mul(eps, r[i]));
}

// s = M r0; delta0 = r.s; NotSpd check; top-of-loop checks for i = 0.
template <int PRE, int FMT, int ND, bool SH>
__global__ void __launch_bounds__(PR, FMT >= 1 ? 8 : 1) k_setup2(Dev D) {
  SG_KERNEL_PROLOGUE
  if (PRE == SG_PRECOND_LEARNED) stage<FMT>(D, T, r0, r1, D.g_offs, D.g_cols, D.g_vals);
  double prs = 0.0;
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const long long i = r0 + (long long)rr * PR + threadIdx.x;
    if (i >= r1) continue;
    const unsigned int m = dmask(D, i, r1, FMT);
    if (!owned(ow, i)) continue;  // ghost rows of s come from the neighbour partitions
    const double si = apply_row<PRE, FMT, ND, SH>(D, T, i, r0, m, D.r0, D.ctl->eps);
    store_s(D, ow, i, si);
    prs += mul(D.r0[i], si);
  }
  if (arrive(D, sys, prs, 0.0, red, &flag)) {
    const double rs = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) { if (D.part) part_fin(D, sys, FIN_SETUP2, rs, 0.0, 0); else fin_setup2(D, sys, rs); }
  }
}

// SPLIT (CSR with scattered columns): d' was written by k_pre_d, so A d' gathers one vector
// instead of forming s + beta d from two gathers per nonzero.
template <int PRE, int FMT, int ND, bool SH, bool SPLIT = false>
__global__ void __launch_bounds__(PR, FMT >= 1 ? 8 : 1) k_iter1(Dev D, int par) {
  SG_KERNEL_PROLOGUE
  const int status = D.st[sys].status;
  if (status == ST_DONE) return;
  const bool run = status == ST_RUN;
  const bool fresh = run ? (D.st[sys].flags & FL_FRESH) != 0 : true;
  const double beta = D.st[sys].beta;
  double* dc = par ? D.d1 : D.d0;
  double* dn = par ? D.d0 : D.d1;
  double* rc = par ? D.r1 : D.r0;
  stage<FMT>(D, T, r0, r1, D.a_offs, D.a_cols, D.a_vals);
  double pdq = 0.0, prr = 0.0;
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const long long i = r0 + (long long)rr * PR + threadIdx.x;
    if (i >= r1) continue;
    const unsigned int m = dmask(D, i, r1, FMT);
    if (run) {
      double dni, qi;
      if (SPLIT) {
        dni = dn[i];
        qi = rowA<FMT, ND, SH, 0>(D, T, i, r0, m, XF{dn, nullptr, 0.0});
      } else {
        dni = add(D.s[i], mul(beta, dc[i]));
        dn[i] = dni;
        qi = rowA<FMT, ND, SH, 1>(D, T, i, r0, m, XF{D.s, dc, beta});
      }
      D.q[i] = qi;
      if (owned(ow, i)) pdq += mul(dni, qi);
    }
    if (fresh) {
      const double rf = sub(D.b[i], rowA<FMT, ND, SH, 0>(D, T, i, r0, m, XF{D.x, nullptr, 0.0}));
      if (run) rc[i] = rf;
      if (owned(ow, i)) prr += mul(rf, rf);
    }
  }
  if (arrive(D, sys, pdq, prr, red, &flag)) {
    double dq, rrf;
    gather_partials2(D, D.sys_blk0, sys, dq, rrf);
    if (threadIdx.x == 0) { if (D.part) part_fin(D, sys, FIN_K1, dq, rrf, run); else fin_k1(D, sys, run, dq, rrf); }
  }
}

// SPLIT: r' was written by k_pre_r (with the x update), so G^T r' gathers one vector.
template <int PRE, int FMT, int ND, bool SH, bool SPLIT = false>
__global__ void __launch_bounds__(PR, FMT >= 1 ? 8 : 1) k_iter2(Dev D, int par) {
  SG_KERNEL_PROLOGUE
  if (D.st[sys].status != ST_RUN) return;
  const double alpha = D.st[sys].alpha;
  const double* dn = par ? D.d0 : D.d1;
  const double* rc = par ? D.r1 : D.r0;
  double* rn = par ? D.r0 : D.r1;
  if (PRE == SG_PRECOND_LEARNED) stage<FMT>(D, T, r0, r1, D.gt_offs, D.gt_cols, D.gt_vals);
  double prr = 0.0;
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const long long i = r0 + (long long)rr * PR + threadIdx.x;
    if (i >= r1) continue;
    const unsigned int m = dmask(D, i, r1, FMT);
    double rni;
    if (SPLIT) {
      rni = rn[i];
    } else {
      D.x[i] = add(D.x[i], mul(alpha, dn[i]));
      rni = sub(rc[i], mul(alpha, D.q[i]));
      rn[i] = rni;
    }
    if (owned(ow, i)) prr += mul(rni, rni);
    if (PRE == SG_PRECOND_LEARNED) {
      if (SPLIT) D.t[i] = rowGt<FMT, ND, SH, 0>(D, T, i, r0, m, XF{rn, nullptr, 0.0});
      else D.t[i] = rowGt<FMT, ND, SH, 2>(D, T, i, r0, m, XF{rc, D.q, alpha});
    }
  }
  if (arrive(D, sys, prr, 0.0, red, &flag)) {
    const double rr = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) { if (D.part) part_fin(D, sys, FIN_RR, rr, 0.0, 0); else fin_rr(D, sys, rr); }
  }
}

// Elementwise halves of K1 / K2 for the SPLIT path: d' = s + beta d; x += alpha d', r' = r - alpha q.
__global__ void __launch_bounds__(PR) k_pre_d(Dev D, int par) {
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  const double beta = D.st[sys].beta;
  const double* dc = par ? D.d1 : D.d0;
  double* dn = par ? D.d0 : D.d1;
  for (long long i = r0 + threadIdx.x; i < r1; i += PR) dn[i] = add(D.s[i], mul(beta, dc[i]));
}

__global__ void __launch_bounds__(PR) k_pre_r(Dev D, int par) {
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  const double alpha = D.st[sys].alpha;
  const double* dn = par ? D.d0 : D.d1;
  const double* rc = par ? D.r1 : D.r0;
  double* rn = par ? D.r0 : D.r1;
  for (long long i = r0 + threadIdx.x; i < r1; i += PR) {
    D.x[i] = add(D.x[i], mul(alpha, dn[i]));
    rn[i] = sub(rc[i], mul(alpha, D.q[i]));
  }
}

__global__ void __launch_bounds__(PR) k_refresh_x(Dev D, int par) {
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  const double alpha = D.st[sys].alpha;
  const double* dn = par ? D.d0 : D.d1;
  const double* xs = (D.st[sys].flags & FL_XINT) ? D.t : D.x;  // x parked in t by a fresh K1
  for (long long i = r0 + threadIdx.x; i < r1; i += PR) D.x[i] = add(xs[i], mul(alpha, dn[i]));
}

// End of a solve with deferred x updates: complete x for systems that stopped with one pending
// (x in t and / or alpha d' not yet added).  Same operations as the deferred kernels would do.
__global__ void __launch_bounds__(PR) k_xflush(Dev D) {
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  const int fl = D.st[sys].flags;
  if (!(fl & (FL_XPEND | FL_XINT))) return;
  const double alpha = D.st[sys].alpha;
  const double* dd = (fl & FL_DPAR) ? D.d0 : D.d1;
  for (long long i = r0 + threadIdx.x; i < r1; i += PR) {
    double v = (fl & FL_XINT) ? D.t[i] : D.x[i];
    if (fl & FL_XPEND) v = add(v, mul(alpha, dd[i]));
    D.x[i] = v;
  }
}

template <int FMT, int ND, bool SH>
__global__ void __launch_bounds__(PR, FMT >= 1 ? 8 : 1) k_refresh_r(Dev D, int par) {
  SG_KERNEL_PROLOGUE
  if (D.st[sys].status != ST_RUN) return;
  double* rn = par ? D.r0 : D.r1;
  stage<FMT>(D, T, r0, r1, D.a_offs, D.a_cols, D.a_vals);
  double prr = 0.0;
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const long long i = r0 + (long long)rr * PR + threadIdx.x;
    if (i >= r1) continue;
    const unsigned int m = dmask(D, i, r1, FMT);
    const double rni = sub(D.b[i], rowA<FMT, ND, SH, 0>(D, T, i, r0, m, XF{D.x, nullptr, 0.0}));
    rn[i] = rni;
    if (owned(ow, i)) prr += mul(rni, rni);
  }
  if (arrive(D, sys, prr, 0.0, red, &flag)) {
    const double rr = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) { if (D.part) part_fin(D, sys, FIN_RR, rr, 0.0, 0); else fin_rr(D, sys, rr); }
  }
}

template <int FMT, int ND, bool SH>
__global__ void __launch_bounds__(PR, FMT >= 1 ? 8 : 1) k_refresh_t(Dev D, int par) {
  SG_KERNEL_PROLOGUE
  if (D.st[sys].status != ST_RUN) return;
  const double* rn = par ? D.r0 : D.r1;
  stage<FMT>(D, T, r0, r1, D.gt_offs, D.gt_cols, D.gt_vals);
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const long long i = r0 + (long long)rr * PR + threadIdx.x;
    if (i >= r1) continue;
    D.t[i] = rowGt<FMT, ND, SH, 0>(D, T, i, r0, dmask(D, i, r1, FMT), XF{rn, nullptr, 0.0});
  }
  (void)red; (void)flag;
}

template <int PRE, int FMT, int ND, bool SH>
__global__ void __launch_bounds__(PR, FMT >= 1 ? 8 : 1) k_iter3(Dev D, int par, int refreshed) {
  SG_KERNEL_PROLOGUE
  if (D.st[sys].status != ST_RUN) return;
  const double* rn = par ? D.r0 : D.r1;
  if (PRE == SG_PRECOND_LEARNED) stage<FMT>(D, T, r0, r1, D.g_offs, D.g_cols, D.g_vals);
  double prs = 0.0;
#pragma unroll
  for (int rr = 0; rr < RPT; ++rr) {
    const long long i = r0 + (long long)rr * PR + threadIdx.x;
    if (i >= r1) continue;
    if (!owned(ow, i)) continue;  // ghost rows of s come from the neighbour partitions
    const unsigned int m = dmask(D, i, r1, FMT);
    const double si = apply_row<PRE, FMT, ND, SH>(D, T, i, r0, m, rn, D.ctl->eps);
    store_s(D, ow, i, si);
    prs += mul(rn[i], si);
  }
  if (arrive(D, sys, prs, 0.0, red, &flag)) {
    const double rs = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) {
      if (D.part) {
        part_fin(D, sys, FIN_K3, rs, 0.0, refreshed);
      } else {
        D.st[sys].flags &= ~(FL_XPEND | FL_XINT | FL_DPAR);  // refresh path: x complete (k_refresh_x)
        fin_k3(D, sys, rs, refreshed);
      }
    }
  }
}

// K2 (SPLIT: r' already written by k_pre_r) for long CSR rows: t = G^T r' from the SELL-32 copy,
// one row per thread in add.at order, 8 products in flight per thread, no row tile (so 4 CTAs
// fit an SM; the generic k_iter2 holds 96 registers).  Same rows, roundings and per-thread
// partials as k_iter2<.., SPLIT>: bit-identical.
__global__ void __launch_bounds__(PR, 4) k_iter2_sell(Dev D, int par) {
  __shared__ double red[PR / 32];
  __shared__ int flag;
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  const double* __restrict__ rn = par ? D.r0 : D.r1;
  double prr = 0.0;
  const long long i = r0 + threadIdx.x;
  if (i < r1) {
    const double rni = rn[i];
    prr = mul(rni, rni);
    const long long b = D.sgt.sbase[i >> 5] + (i & 31);
    const int len = D.sgt.offs[i + 1] - D.sgt.offs[i];
    const double* __restrict__ sv = D.sgt.vals + b;
    const int32_t* __restrict__ sc = D.sgt.cols + b;
    double s = 0.0;
    int k = 0;
    for (; k + 8 <= len; k += 8) {
      int c[8];
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) c[u] = __ldg(sc + 32 * (k + u));
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = mul(__ldg(sv + 32 * (k + u)), __ldg(rn + c[u]));
#pragma unroll
      for (int u = 0; u < 8; ++u) s = add(s, v[u]);
    }
    for (; k < len; ++k) s = add(s, mul(__ldg(sv + 32 * k), __ldg(rn + __ldg(sc + 32 * k))));
    D.t[i] = s;
  }
  if (arrive(D, sys, prr, 0.0, red, &flag)) {
    const double rr = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) fin_rr(D, sys, rr);
  }
}

// K3 for long CSR rows of G (C4: ~420 per row on the A^2 pattern): one warp per row in numpy's
// exact pairwise order (warp_row_numpy), coalesced instead of one thread walking each row.  The
// CTA keeps k_iter3's rows and its per-thread r.s partials (one row per thread slot), so the
// result, the partial sums and the finaliser are bit-identical to k_iter3's.
__global__ void __launch_bounds__(PR) k_iter3_wr(Dev D, int par, int refreshed) {
  __shared__ double red[PR / 32];
  __shared__ int flag;
  __shared__ int2 leaf[PR / 32][kWarpLeaves];
  __shared__ double lsum[PR / 32][kWarpLeaves];
  __shared__ double prow[PR];
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  const double* rn = par ? D.r0 : D.r1;
  const double eps = D.ctl->eps;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long i = r0 + w; i < r1; i += PR / 32) {
    const double y = warp_row_numpy<0>(D.g_vals, D.g_cols, D.g_offs[i], D.g_offs[i + 1],
                                       XF{D.t, nullptr, 0.0}, leaf[w], lsum[w]);
    if (lane == 0) {
      const double ri = rn[i];
      const double si = add(y, mul(eps, ri));
      D.s[i] = si;
      prow[i - r0] = mul(ri, si);
    }
  }
  __syncthreads();
  const double prs = r0 + threadIdx.x < r1 ? prow[threadIdx.x] : 0.0;
  if (arrive(D, sys, prs, 0.0, red, &flag)) {
    const double rs = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) fin_k3(D, sys, rs, refreshed);
  }
}

// ------------------------------------------------------------------ small systems: one CTA / cluster per system
// For stencil (DIA) systems of <= kSmallRows rows the multi-kernel iteration is launch- and
// latency-bound (~18-19 us per iteration from 256 to 8100 rows).  Measured per iteration, one
// CTA / multi-kernel: 256 rows 8.0 / 18.0 us, 1024 rows 9.4 / 19.4, 2304 rows 13.0 / 18.2,
// 4096 rows 19.0 / 18.9, 8100 rows 31.5 / 19.2 (profiles/small_probe.py).  One 1024-thread CTA runs whole
// iterations of ONE system with CTA barriers between the phases instead of kernel boundaries:
// the same phases, roundings, summation orders and finalisers as k_iter1/2/3 + k_refresh_*
// (dot products: per-thread partials in row order, then the block tree).  `iters` iterations per
// launch (the host polls the active count between launches, as between graph chunks).
//
// Mid-size systems (up to kClusterRows rows) run the same loop on a THREAD-BLOCK CLUSTER of CN
// CTAs (one per SM, CN <= 16): rows interleave over the cluster's CN * 1024 threads, the phase
// barriers are hardware cluster barriers (barrier.cluster release / acquire: every global write
// of a phase is visible to the whole cluster after it) and the dot products add the CTAs' block
// sums in rank order through distributed shared memory (rank 0's slots), so one launch still runs
// whole iterations with no kernel boundary.
constexpr int kSmallRows = 3072;
constexpr int kSmallThreads = 1024;
#ifndef SG_CLUSTER_ROWS
#define SG_CLUSTER_ROWS 32768
#endif
constexpr int kClusterRows = SG_CLUSTER_ROWS;

template <int CN>
__device__ __forceinline__ void sm_sync() {
  if constexpr (CN == 1) __syncthreads();
  else asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// The system's dot product: block tree per CTA, then (CN > 1) rank 0 adds the CTAs' sums in rank
// order from its shared-memory slots (written by the ranks through DSMEM).  Valid in thread 0 of
// rank 0 after the call; `slots` is a __shared__ [2][16] array used alternately by consecutive
// calls (`seq` counts them), so a rank's next write never meets rank 0 still reading.
template <int CN>
__device__ __forceinline__ double sm_sum(double v, double* red, double* slots_all, int& seq) {
  const double bs = block_sum(v, red);
  if constexpr (CN == 1) {
    return bs;
  } else {
    double* slots = slots_all + 16 * (seq++ & 1);
    if (threadIdx.x == 0) {
      uint32_t dst;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(dst) : "r"(smem_u32(slots + cluster_rank())));
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dst), "d"(bs) : "memory");
    }
    sm_sync<CN>();
    double r = 0.0;
    if (threadIdx.x == 0 && cluster_rank() == 0)
      for (int k = 0; k < CN; ++k) r += slots[k];
    return r;
  }
}

template <int PRE, int FMT, int ND, int CN = 1>
__global__ void __launch_bounds__(kSmallThreads, 1) k_pcg_small(Dev D, int iters, long long period) {
  __shared__ double red[32];
  __shared__ double slots[32];
  int seq = 0;
  const int rank = CN == 1 ? 0 : (int)cluster_rank();
  const int sys = blockIdx.x / CN, tid = rank * kSmallThreads + (int)threadIdx.x;
  constexpr int NT = CN * kSmallThreads;  // threads per system
  const bool lead = threadIdx.x == 0 && rank == 0;
  const long long s0 = D.blk_r0[D.sys_blk0[sys]], s1 = D.sys_r1[sys];
  const double eps = D.ctl->eps;
  double* x = D.x;
  double* r = D.r0;
  double* d = D.d0;
  auto rowA = [&](long long i, const XF& f) {
    const unsigned int m = D.dia.mask[i];
    return FMT == 2 ? dia_row_numpy_sym<ND, 0>(D.dia, D.dia.av, (int)i, m, f)
                    : dia_row_numpy<ND, 0>(D.dia, D.dia.av, (int)i, m, f);
  };
  for (int c = 0; c < iters; ++c) {
    SysState& S = D.st[sys];
    const int status = S.status;
    if (status == ST_DONE) break;
    const bool run = status == ST_RUN;
    const bool fresh = run ? (S.flags & FL_FRESH) != 0 : true;
    const bool refresh = run && S.i > 0 && S.i % period == 0;
    const double beta = S.beta;
    // K1: d = s + beta d; q = A d, d.q; fresh residual b - A x (pcg.py:176-184, 208-215)
    double pdq = 0.0, prr = 0.0;
    if (run) {
      for (long long i = s0 + tid; i < s1; i += NT) d[i] = add(D.s[i], mul(beta, d[i]));
      sm_sync<CN>();
      for (long long i = s0 + tid; i < s1; i += NT) {
        const double qi = rowA(i, XF{d, nullptr, 0.0});
        D.q[i] = qi;
        pdq += mul(d[i], qi);
      }
    }
    if (fresh) {
      for (long long i = s0 + tid; i < s1; i += NT) {
        const double rf = sub(D.b[i], rowA(i, XF{x, nullptr, 0.0}));
        if (run) r[i] = rf;
        prr += mul(rf, rf);
      }
    }
    const double dq = sm_sum<CN>(pdq, red, slots, seq);
    const double rrf = sm_sum<CN>(prr, red, slots, seq);
    if (lead) fin_k1(D, sys, run, dq, rrf);
    sm_sync<CN>();
    if (S.status != ST_RUN) continue;
    const double alpha = S.alpha;
    // K2: x += alpha d; r -= alpha q (or, on refresh iterations, r = b - A x); ||r||^2
    double prn = 0.0;
    for (long long i = s0 + tid; i < s1; i += NT) x[i] = add(x[i], mul(alpha, d[i]));
    if (refresh) {
      sm_sync<CN>();
      for (long long i = s0 + tid; i < s1; i += NT) {
        const double rn = sub(D.b[i], rowA(i, XF{x, nullptr, 0.0}));
        r[i] = rn;
        prn += mul(rn, rn);
      }
    } else {
      for (long long i = s0 + tid; i < s1; i += NT) {
        const double rn = sub(r[i], mul(alpha, D.q[i]));
        r[i] = rn;
        prn += mul(rn, rn);
      }
    }
    const double rr = sm_sum<CN>(prn, red, slots, seq);
    if (lead) fin_rr(D, sys, rr);
    sm_sync<CN>();
    // K3: s = M r (learned: t = G^T r, then s = G t + eps r); r.s -- the preconditioner apply,
    // timed by the lead thread between the phase barriers (the reference's t_apply)
    unsigned long long ta = 0;
    if (lead) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ta));
    if (PRE == SG_PRECOND_LEARNED) {
      for (long long i = s0 + tid; i < s1; i += NT)
        D.t[i] = dia_row_t_seq<ND, 0>(D.dia, D.dia.gv, (int)i, D.dia.mask[i], XF{r, nullptr, 0.0});
      sm_sync<CN>();
    }
    double prs = 0.0;
    for (long long i = s0 + tid; i < s1; i += NT) {
      double si;
      if (PRE == SG_PRECOND_IDENTITY) si = r[i];
      else if (PRE == SG_PRECOND_JACOBI) si = mul(r[i], D.inv_diag[i]);
      else si = add(dia_row_numpy<ND, 0>(D.dia, D.dia.gv, (int)i, D.dia.mask[i], XF{D.t, nullptr, 0.0}),
                    mul(eps, r[i]));
      D.s[i] = si;
      prs += mul(r[i], si);
    }
    const double rs = sm_sum<CN>(prs, red, slots, seq);
    if (lead) {
      unsigned long long tb;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb));
      atomicAdd(&D.ctl->apply_ns, tb - ta);
      fin_k3(D, sys, rs, refresh ? 1 : 0);
    }
    sm_sync<CN>();
  }
}

// ------------------------------------------------------------------ small systems, shared-memory resident
// The same iteration as k_pcg_small with the whole system held in shared memory: a cluster of CN
// CTAs (CN = 1 .. 16) splits the system into CN blocks of R consecutive rows; each CTA keeps its
// rows of x, r, d, q, s, t, b, its mask bytes, and A's / G's diagonals on its rows +- H (the
// mirror entries of the neighbour rows), loaded once per launch and written back at its end.  A
// neighbour row of another CTA is read from that CTA's shared memory through DSMEM
// (ld.shared::cluster; H <= R, so only ranks +-1).  Fewer barriers per iteration than the
// global-memory loop: d' = s + beta d and r' = r - alpha q of NEIGHBOUR rows are recomputed where
// q = A d' and t = G^T r' need them (bitwise the stored values), the own rows' d', r' wait in
// registers until the next barrier; the dot products are cluster all-reduces (every rank adds
// the ranks' block sums in rank order: identical values everywhere), so every CTA runs the
// finalisers on its own copy of the system state and only rank 0 reports (history, active
// count).  Three cluster barriers per iteration (five on refresh iterations).  Roundings,
// summation orders and finalisers are k_pcg_small's.
struct SmemSys {
  double *x, *r, *d, *q, *s, *t, *b;  // [R] own rows
  double* ae;                         // [NA][R + 2H] A's diagonals, rows a0 - H ..
  double* ge;                         // [ND][R + 2H] G's diagonals
  unsigned char* mk;                  // [R]
};

__host__ __device__ constexpr size_t smem_sys_bytes(int R, int H, int NA, int ND) {
  return ((size_t)7 * R + (size_t)(NA + ND) * (R + 2 * H)) * 8 + (size_t)(R + 15) / 16 * 16;
}

__device__ __forceinline__ double ld_peer(const double* local, int rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(local)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}

// Vector value at system row j (0 outside the system: such entries are masked out anyway).
template <int CN>
__device__ __forceinline__ double vsm(const double* v, long long j, long long s0, long long s1, long long a0, int R,
                                      int rank) {
  if (j < s0 || j >= s1) return 0.0;
  const int li = (int)(j - a0);
  if (CN > 1 && li < 0) return ld_peer(v + li + R, rank - 1);
  if (CN > 1 && li >= R) return ld_peer(v + li - R, rank + 1);
  return v[li];
}

// Two dot products at once: block trees per CTA, then (CN > 1) every rank's thread 0 stores its
// block sums into every rank's slots and, after the cluster barrier, adds them in rank order.
// Valid in thread 0 of every CTA.  slots: __shared__ [2 parities][2][16].
template <int CN>
__device__ __forceinline__ void sm_allreduce2(double a, double b, double* red, double* slots_all, int& seq, double& ra,
                                              double& rb) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) { red[wid] = a; red[32 + wid] = b; }
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double xa = 0.0, xb = 0.0;
  if (wid == 0) {
    xa = warp_sum(lane < nw ? red[lane] : 0.0);
    xb = warp_sum(lane < nw ? red[32 + lane] : 0.0);
  }
  if constexpr (CN == 1) {
    ra = xa;
    rb = xb;
  } else {
    double* slots = slots_all + 32 * (seq++ & 1);
    const int rank = (int)cluster_rank();
    if (threadIdx.x == 0)
      for (int k = 0; k < CN; ++k) {
        uint32_t pa, pb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(pa) : "r"(smem_u32(slots + rank)), "r"(k));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(pb) : "r"(smem_u32(slots + 16 + rank)), "r"(k));
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(pa), "d"(xa) : "memory");
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(pb), "d"(xb) : "memory");
      }
    sm_sync<CN>();
    ra = 0.0;
    rb = 0.0;
    if (threadIdx.x == 0)
      for (int k = 0; k < CN; ++k) { ra += slots[k]; rb += slots[16 + k]; }
  }
}

template <int PRE, int FMT, int ND, int CN>
__global__ void __launch_bounds__(kSmallThreads, 1) k_pcg_smem(Dev D, int iters, long long period, int R) {
  constexpr int NA = FMT == 2 ? ND / 2 + 1 : ND;
  constexpr int RPT = 2;  // R <= 2 * kSmallThreads
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ double red[64];
  __shared__ double slots[64];
  __shared__ __align__(16) SysState SS;  // this CTA's copy of the system state
  int seq = 0;
  const int rank = CN == 1 ? 0 : (int)cluster_rank();
  const int sys = blockIdx.x / CN, tid = threadIdx.x;
  const bool pri = rank == 0;
  const long long s0 = D.blk_r0[D.sys_blk0[sys]], s1 = D.sys_r1[sys];
  const int H = D.dia.halo, RE = R + 2 * H;
  const long long a0 = s0 + (long long)rank * R;
  const int Rown = (int)(a0 >= s1 ? 0 : (s1 - a0 < R ? s1 - a0 : R));
  const double eps = D.ctl->eps;
  SmemSys M;
  {
    double* p = reinterpret_cast<double*>(smraw);
    M.x = p; M.r = p + R; M.d = p + 2 * R; M.q = p + 3 * R; M.s = p + 4 * R; M.t = p + 5 * R; M.b = p + 6 * R;
    M.ae = p + 7 * R;
    M.ge = M.ae + NA * RE;
    M.mk = reinterpret_cast<unsigned char*>(M.ge + ND * RE);
  }
  int off[ND], mir[ND];
#pragma unroll
  for (int dg = 0; dg < ND; ++dg) { off[dg] = D.dia.off[dg]; mir[dg] = D.dia.mir[dg]; }
  // load: own rows of the vectors, the diagonals on rows a0 - H .. a0 + R + H (zero outside)
  for (int li = tid; li < R; li += kSmallThreads) {
    const bool in = li < Rown;
    const long long i = a0 + li;
    M.x[li] = in ? D.x[i] : 0.0;
    M.r[li] = in ? D.r0[i] : 0.0;
    M.d[li] = in ? D.d0[i] : 0.0;
    M.s[li] = in ? D.s[i] : 0.0;
    M.b[li] = in ? D.b[i] : 0.0;
    M.q[li] = 0.0;
    M.t[li] = 0.0;
    M.mk[li] = in ? D.dia.mask[i] : (unsigned char)0;
  }
  for (int e = tid; e < RE; e += kSmallThreads) {
    const long long i = a0 - H + e;
    const bool in = i >= s0 && i < s1;
#pragma unroll
    for (int dg = 0; dg < NA; ++dg) M.ae[dg * RE + e] = in ? D.dia.av[dg][i] : 0.0;
    if (PRE == SG_PRECOND_LEARNED)
#pragma unroll
      for (int dg = 0; dg < ND; ++dg) M.ge[dg * RE + e] = in ? D.dia.gv[dg][i] : 0.0;
  }
  if (tid == 0) SS = D.st[sys];
  sm_sync<CN>();
  auto Aval = [&](int li, int dg) {
    const int e = li + H;
    return (FMT == 2 && off[dg] > 0) ? M.ae[mir[dg] * RE + e + off[dg]] : M.ae[dg * RE + e];
  };
  auto V = [&](const double* v, long long j) { return vsm<CN>(v, j, s0, s1, a0, R, rank); };
  // b - A x (x of the neighbours as stored)
  auto resid = [&](int li) {
    const long long j = a0 + li;
    double p[ND];
#pragma unroll
    for (int dg = 0; dg < ND; ++dg) p[dg] = mul(Aval(li, dg), V(M.x, j + off[dg]));
    return sub(M.b[li], combine_numpy<ND>(p, M.mk[li]));
  };
  for (int c = 0; c < iters; ++c) {
    const int status = SS.status;
    if (status == ST_DONE) break;
    const bool run = status == ST_RUN;
    const bool fresh = run ? (SS.flags & FL_FRESH) != 0 : true;
    const bool refresh = run && SS.i > 0 && SS.i % period == 0;
    const double beta = SS.beta;
    // K1: q = A d' with d' = s + beta d recomputed for the neighbour rows; fresh residual
    double pdq = 0.0, prr = 0.0, dn[RPT];
#pragma unroll
    for (int h = 0; h < RPT; ++h) {
      const int li = tid + h * kSmallThreads;
      dn[h] = 0.0;
      if (li < Rown) {
        const long long j = a0 + li;
        if (run) {
          double p[ND];
#pragma unroll
          for (int dg = 0; dg < ND; ++dg) {
            const long long jj = j + off[dg];
            const double dj = add(V(M.s, jj), mul(beta, V(M.d, jj)));
            p[dg] = mul(Aval(li, dg), dj);
          }
          const double qi = combine_numpy<ND>(p, M.mk[li]);
          dn[h] = add(M.s[li], mul(beta, M.d[li]));
          M.q[li] = qi;
          pdq += mul(dn[h], qi);
        }
        if (fresh) {
          const double rf = resid(li);
          if (run) M.r[li] = rf;
          prr += mul(rf, rf);
        }
      }
    }
    double dq, rrf;
    sm_allreduce2<CN>(pdq, prr, red, slots, seq, dq, rrf);  // cluster barrier: every d read is done
    if (run)
#pragma unroll
      for (int h = 0; h < RPT; ++h)
        if (tid + h * kSmallThreads < Rown) M.d[tid + h * kSmallThreads] = dn[h];
    if (tid == 0) fin_k1_s(D, SS, sys, run, dq, rrf, pri);
    __syncthreads();
    if (SS.status != ST_RUN) continue;
    const double alpha = SS.alpha;
    unsigned long long ta = 0;
    if (tid == 0 && pri) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ta));
    double prn = 0.0;
    if (!refresh) {
      // x += alpha d'; r' = r - alpha q (own rows in registers); t = G^T r' with the neighbours'
      // r' recomputed from their r and q (q of every row is final since the all-reduce barrier)
      double rn[RPT];
#pragma unroll
      for (int h = 0; h < RPT; ++h) {
        const int li = tid + h * kSmallThreads;
        rn[h] = 0.0;
        if (li < Rown) {
          const long long j = a0 + li;
          M.x[li] = add(M.x[li], mul(alpha, M.d[li]));
          rn[h] = sub(M.r[li], mul(alpha, M.q[li]));
          prn += mul(rn[h], rn[h]);
          if (PRE == SG_PRECOND_LEARNED) {
            const int e = li + H;
            double p[ND];
#pragma unroll
            for (int dg = 0; dg < ND; ++dg) {
              const long long jj = j + off[dg];
              const double rj = sub(V(M.r, jj), mul(alpha, V(M.q, jj)));
              p[dg] = mul(M.ge[mir[dg] * RE + e + off[dg]], rj);
            }
            M.t[li] = combine_seq<ND>(p, M.mk[li]);
          }
        }
      }
      sm_sync<CN>();  // every r and t read / write of the phase is done
#pragma unroll
      for (int h = 0; h < RPT; ++h)
        if (tid + h * kSmallThreads < Rown) M.r[tid + h * kSmallThreads] = rn[h];
      if (PRE != SG_PRECOND_LEARNED) __syncthreads();
    } else {
      // refresh iteration (every `period`): r = b - A x needs the neighbours' new x first
      for (int li = tid; li < Rown; li += kSmallThreads) M.x[li] = add(M.x[li], mul(alpha, M.d[li]));
      sm_sync<CN>();
      for (int li = tid; li < Rown; li += kSmallThreads) {
        const double rv = resid(li);
        M.r[li] = rv;
        prn += mul(rv, rv);
      }
      sm_sync<CN>();
      if (PRE == SG_PRECOND_LEARNED) {
        for (int li = tid; li < Rown; li += kSmallThreads) {
          const long long j = a0 + li;
          const int e = li + H;
          double p[ND];
#pragma unroll
          for (int dg = 0; dg < ND; ++dg) p[dg] = mul(M.ge[mir[dg] * RE + e + off[dg]], V(M.r, j + off[dg]));
          M.t[li] = combine_seq<ND>(p, M.mk[li]);
        }
        sm_sync<CN>();
      }
    }
    // K3: s = M r' (learned: s = G t + eps r'); r'.s
    double prs = 0.0;
    for (int li = tid; li < Rown; li += kSmallThreads) {
      double si;
      if (PRE == SG_PRECOND_IDENTITY) si = M.r[li];
      else if (PRE == SG_PRECOND_JACOBI) si = mul(M.r[li], D.inv_diag[a0 + li]);
      else {
        const long long j = a0 + li;
        const int e = li + H;
        double p[ND];
#pragma unroll
        for (int dg = 0; dg < ND; ++dg) p[dg] = mul(M.ge[dg * RE + e], V(M.t, j + off[dg]));
        si = add(combine_numpy<ND>(p, M.mk[li]), mul(eps, M.r[li]));
      }
      M.s[li] = si;
      prs += mul(M.r[li], si);
    }
    double rr, rs;
    sm_allreduce2<CN>(prn, prs, red, slots, seq, rr, rs);
    if (tid == 0) {
      if (pri) {
        unsigned long long tb;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb));
        atomicAdd(&D.ctl->apply_ns, tb - ta);
      }
      SS.rr = rr;
      fin_k3_s(D, SS, sys, rs, refresh ? 1 : 0, pri);
    }
    __syncthreads();
  }
  // write back the state the next launch (and the caller) reads
  if (tid == 0 && pri) D.st[sys] = SS;
  for (int li = tid; li < Rown; li += kSmallThreads) {
    const long long i = a0 + li;
    D.x[i] = M.x[li];
    D.r0[i] = M.r[li];
    D.d0[i] = M.d[li];
    D.s[i] = M.s[li];
    D.q[i] = M.q[li];
    D.t[i] = M.t[li];
  }
  sm_sync<CN>();  // no CTA leaves while a peer may still read its shared memory
}

// ------------------------------------------------------------------ halo-staged DIA kernels
// For stencil patterns with a small halo H = max |offset| the neighbour values a row needs are
// staged once per tile in shared memory (tile +- H rows, computed on the fly from their inputs)
// instead of being re-read / re-derived per neighbour.  That turns K2 + K3 into ONE kernel:
//   r' = r - alpha q over tile +- 2H  ->  t = G^T r' over tile +- H  ->  s = G t + eps r'
// so t never goes to HBM and G is streamed once per iteration instead of twice.  Every value is
// computed with the same roundings and summation order as the unstaged kernels (bit-identical
// results); rows outside the tile's system stage as 0 and are never selected by the masks.
__device__ __forceinline__ void sys_bounds(const Dev& D, int sys, long long& s0, long long& s1) {
  s0 = D.blk_r0[D.sys_blk0[sys]];
  s1 = D.sys_r1[sys];
}

// numpy-order row of A / G with the neighbour values taken from shared memory (xs[li + off]).
template <int FMT, int ND>
__device__ __forceinline__ double dia_row_sm(const Dia& dd, const double* const* Vd, int i, int li,
                                             unsigned int m, const double* xs) {
  constexpr int NA = ND > 0 ? ND : 1;
  double a[NA], p[NA];
#pragma unroll
  for (int d = 0; d < ND; ++d)
    a[d] = (FMT == 2 && dd.off[d] > 0) ? __ldg(Vd[dd.mir[d]] + i + dd.off[d]) : __ldg(Vd[d] + i);
#pragma unroll
  for (int d = 0; d < ND; ++d) p[d] = mul(a[d], xs[li + dd.off[d]]);
  return combine_numpy<NA>(p, m);
}

// Clamp a neighbour row into the tile's system: staged loads are issued unconditionally (all of
// a thread's loads in flight at once) and the out-of-system values are replaced by 0 afterwards.
__device__ __forceinline__ long long clampr(long long j, long long s0, long long s1) {
  return j < s0 ? s0 : (j >= s1 ? s1 - 1 : j);
}

// K1 with d' staged: d'[j] = s[j] + beta d[j] for j in tile +- H, then q = A d'.
// NH = ceil(H / PR) fixes the trip counts of the staging loops.
template <int FMT, int ND, int NH, bool PART = false>
__global__ void __launch_bounds__(PR, 6) k_iter1_st(Dev D, int par) {
  extern __shared__ double sm[];
  __shared__ double red[PR / 32];
  __shared__ int flag;
  int sys; long long r0, r1, s0, s1;
  block_rows(D, sys, r0, r1);
  const int status = D.st[sys].status;
  if (status == ST_DONE) return;
  sys_bounds(D, sys, s0, s1);
  const Own ow = own_get<PART>(D, sys);
  const bool run = status == ST_RUN;
  const bool fresh = run ? (D.st[sys].flags & FL_FRESH) != 0 : true;
  const double beta = D.st[sys].beta;
  const double* dc = par ? D.d1 : D.d0;
  double* dn = par ? D.d0 : D.d1;
  double* rc = par ? D.r1 : D.r0;
  const int H = D.dia.halo;
  const long long lo = r0 - H;
  double pdq = 0.0, prr = 0.0;
  if (run) {
    constexpr int NJ = kRpt + 2 * NH;
    const int span = (int)(r1 - r0) + 2 * H;
    double sv[NJ], dv[NJ];
#pragma unroll
    for (int k = 0; k < NJ; ++k) {
      const long long jc = clampr(lo + k * PR + threadIdx.x, s0, s1);
      sv[k] = __ldg(D.s + jc);
      dv[k] = __ldg(dc + jc);
    }
#pragma unroll
    for (int k = 0; k < NJ; ++k) {
      const int lj = k * PR + threadIdx.x;
      if (lj < span) {
        const long long j = lo + lj;
        double v = 0.0;
        if (j >= s0 && j < s1) {
          v = add(sv[k], mul(beta, dv[k]));
          if (j >= r0 && j < r1) dn[j] = v;
        }
        sm[lj] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < kRpt; ++rr) {
      const long long i = r0 + (long long)rr * PR + threadIdx.x;
      if (i >= r1) continue;
      const int li = (int)(i - lo);
      const double qi = dia_row_sm<FMT, ND>(D.dia, D.dia.av, (int)i, li, D.dia.mask[i], sm);
      D.q[i] = qi;
      if (owned(ow, i)) pdq += mul(sm[li], qi);
    }
  }
  if (fresh) {
#pragma unroll
    for (int rr = 0; rr < kRpt; ++rr) {
      const long long i = r0 + (long long)rr * PR + threadIdx.x;
      if (i >= r1) continue;
      const unsigned int m = D.dia.mask[i];
      const double ax = FMT == 2 ? dia_row_numpy_sym<ND, 0>(D.dia, D.dia.av, (int)i, m, XF{D.x, nullptr, 0.0})
                                 : dia_row_numpy<ND, 0>(D.dia, D.dia.av, (int)i, m, XF{D.x, nullptr, 0.0});
      const double rf = sub(D.b[i], ax);
      if (run) rc[i] = rf;
      if (owned(ow, i)) prr += mul(rf, rf);
    }
  }
  if (arrive(D, sys, pdq, prr, red, &flag)) {
    double dq, rrf;
    gather_partials2(D, D.sys_blk0, sys, dq, rrf);
    if (threadIdx.x == 0) { if (PART) part_fin(D, sys, FIN_K1, dq, rrf, run); else fin_k1(D, sys, run, dq, rrf); }
  }
}

// K2 + K3 fused (learned preconditioner, non-refresh iterations).
//   sr[j - (r0-2H)] = r'[j] = r[j] - alpha q[j]   j in tile +- 2H
//   st[j - (r0-H)]  = t[j]  = (G^T r')[j]          j in tile +- H
//   s[i] = G t + eps r'                             own rows;  partials ||r'||^2, r'.s
template <int ND, int NH, bool PART = false>
__global__ void __launch_bounds__(PR, 5) k_iter23_st(Dev D, int par) {
  extern __shared__ double sm[];
  __shared__ double red[PR / 32];
  __shared__ int flag;
  int sys; long long r0, r1, s0, s1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  sys_bounds(D, sys, s0, s1);
  const Own ow = own_get<PART>(D, sys);
  const double alpha = D.st[sys].alpha;
  const double eps = D.ctl->eps;
  const double* dn = par ? D.d0 : D.d1;
  const double* rc = par ? D.r1 : D.r0;
  double* rn = par ? D.r0 : D.r1;
  const int H = D.dia.halo;
  const int T = (int)(r1 - r0);
  double* sr = sm;                      // T + 4H
  double* st = sm + T + 4 * H;          // T + 2H
  const long long lo2 = r0 - 2 * H, lo1 = r0 - H;
  // halo rows of r' (below and above the tile): loads first
  constexpr int NK = 4 * NH;
  double hr[NK], hq[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int idx = k * PR + threadIdx.x;
    const long long j = idx < 2 * H ? lo2 + idx : r1 + (idx - 2 * H);
    const long long jc = clampr(j, s0, s1);
    hr[k] = __ldg(rc + jc);
    hq[k] = __ldg(D.q + jc);
  }
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const int idx = k * PR + threadIdx.x;
    if (idx < 4 * H) {
      const long long j = idx < 2 * H ? lo2 + idx : r1 + (idx - 2 * H);
      sr[j - lo2] = (j >= s0 && j < s1) ? sub(hr[k], mul(alpha, hq[k])) : 0.0;
    }
  }
  // own rows: r', x, ||r'||^2 (same per-thread row order as k_iter2)
  double prr = 0.0, prs = 0.0;
#pragma unroll
  for (int rr = 0; rr < kRpt; ++rr) {
    const long long i = r0 + (long long)rr * PR + threadIdx.x;
    if (i >= r1) continue;
    D.x[i] = add(D.x[i], mul(alpha, dn[i]));
    const double rni = sub(rc[i], mul(alpha, D.q[i]));
    rn[i] = rni;
    sr[i - lo2] = rni;
    if (owned(ow, i)) prr += mul(rni, rni);
  }
  __syncthreads();
  // t = G^T r' over tile +- H (add.at order; G^T row j on diagonal d = G's mirror at j + off),
  // two rows per thread per batch with all their loads in flight
  constexpr int NJ = kRpt + 2 * NH;
  const int span = T + 2 * H;
#pragma unroll
  for (int kb = 0; kb < NJ; kb += 2) {
    double a[2][ND];
    unsigned int m[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long jc = clampr(lo1 + (kb + u) * PR + threadIdx.x, s0, s1);
      m[u] = D.dia.mask[jc];
#pragma unroll
      for (int d = 0; d < ND; ++d) a[u][d] = __ldg(D.dia.gv[D.dia.mir[d]] + jc + D.dia.off[d]);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int lj1 = (kb + u) * PR + threadIdx.x;
      if (kb + u < NJ && lj1 < span) {
        const long long j = lo1 + lj1;
        double v = 0.0;
        if (j >= s0 && j < s1) {
          const int lj = lj1 + H;  // index of row j in sr
#pragma unroll
          for (int d = 0; d < ND; ++d)
            if (m[u] & (1u << d)) v = add(v, mul(a[u][d], sr[lj + D.dia.off[d]]));
        }
        st[lj1] = v;
      }
    }
  }
  __syncthreads();
  // s = G t + eps r'
#pragma unroll
  for (int rr = 0; rr < kRpt; ++rr) {
    const long long i = r0 + (long long)rr * PR + threadIdx.x;
    if (i >= r1 || !owned(ow, i)) continue;
    const double y = dia_row_sm<1, ND>(D.dia, D.dia.gv, (int)i, (int)(i - lo1), D.dia.mask[i], st);
    const double rni = sr[i - lo2];
    const double si = add(y, mul(eps, rni));
    store_s(D, ow, i, si);
    prs += mul(rni, si);
  }
  if (arrive(D, sys, prr, prs, red, &flag)) {
    double rr, rs;
    gather_partials2(D, D.sys_blk0, sys, rr, rs);
    if (threadIdx.x == 0) {
      if (PART) {
        part_fin(D, sys, FIN_K23, rr, rs, 0);
      } else {
        D.st[sys].rr = rr;
        fin_k3(D, sys, rs, 0);
      }
    }
  }
}


// ------------------------------------------------------------------ sliding-window K2 + K3
// The same fused K2 + K3 as k_iter23_st, organised as a stream instead of independent tiles: a
// CTA walks a RANGE of rows (inside one system) in chunks of C = kSwC rows.  The bulk-copy
// engine (cp.async.bulk + mbarrier) streams each chunk's r, q, G diagonals and mask (the "lead"
// chunk, 2*NH chunks ahead of the output) plus the x, d rows of the output chunk into shared
// memory one chunk ahead of the compute.  Per step k:
//   A  r' = r - alpha q             lead chunk k        (own rows: r' to HBM, ||r'||^2)
//   B  t  = G^T r'                  chunk k - NH        (G, r' of chunks k-2NH .. k)
//   C  s  = G t + eps r', x += alpha d   chunk k - 2NH  (r'.s)
// G, the mask, r' and t live in power-of-two RING-row rings indexed by (row - LB) & (RING-1), so
// a neighbour access is one add, one and, one shared load; the diagonal set is symmetric and
// sorted, so the mirror of diagonal d is ND-1-d at compile time.  Every byte of A's / G's / the
// vectors' rows is read from HBM once per iteration (plus a 4*NH-chunk halo at the two ends of a
// range).  Results are bit-identical to k_iter2 + k_iter3 except for the order of the two dot
// products' partial sums (per range instead of per tile).
__host__ __device__ constexpr int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

template <int ND, int NH>
struct Sw23 {
  static constexpr int C = kSwC;
  static constexpr int P = 3;              // chunks in flight (incl. the current one)
  static constexpr int NG = P + 2 * NH;    // ring chunks of G, mask and r' (r lands in place)
  static constexpr int NT = 2 * NH + 1;    // ring chunks of t
  static constexpr int GR = NG * C, TR = NT * C;
  // bytes: G [ND][GR] | r' [GR] | t [TR] | q staging [P][C] | mask [GR]
  static constexpr size_t SMEM = (size_t)(ND + 1) * GR * 8 + (size_t)TR * 8 + (size_t)P * C * 8 + GR;
};

// Ring index of a neighbour: base + tid + off lies within one ring length of [0, R).
__device__ __forceinline__ int ring_wrap(int x, int R) {
  x = x < 0 ? x + R : x;
  return x >= R ? x - R : x;
}

// The same for neighbour d of a sorted, symmetric diagonal set with an odd count (ND 5, 7):
// offsets below the middle are negative, above it positive, the middle one is 0 -- so one
// wrap test (or none) per diagonal.  Even ND (padded sets) keep the two-sided wrap.
template <int ND>
__device__ __forceinline__ int ring_nb(int base, const int (&off)[ND], int d, int R) {
  if constexpr (ND % 2 == 1) {
    if (d == ND / 2) return base;
    const int x = base + off[d];
    if (d < ND / 2) return x < 0 ? x + R : x;
    return x >= R ? x - R : x;
  } else {
    return ring_wrap(base + off[d], R);
  }
}

// Warp-specialised: warps 0..7 compute (one row per thread per phase, named barrier 1 between
// phases), warp 8 only drives the bulk-copy engine -- it refills a ring slot as soon as the
// consumers' `empty` barrier says the step that last used it is done, so no copy issue ever
// sits on the consumers' critical path between their barriers.
constexpr int kSwThreads = PR + 32;

template <int ND, int NH, bool PART = false>
__global__ void __launch_bounds__(kSwThreads, 3) k_iter23_sw(Dev D, int par) {
  using G = Sw23<ND, NH>;
  constexpr int C = G::C, P = G::P, NG = G::NG, NT = G::NT, GR = G::GR, TR = G::TR;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bars[P];
  __shared__ __align__(8) uint64_t empty[P];
  __shared__ double red[kSwThreads / 32];
  __shared__ int flag;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int sys = D.rng_sys[b];
  if (D.st[sys].status != ST_RUN) return;
  long long s0, s1;
  sys_bounds(D, sys, s0, s1);
  const long long R0 = D.rng_r0[b];
  const long long R1 = R0 + D.rng_len < s1 ? R0 + D.rng_len : s1;
  const double alpha = D.st[sys].alpha;
  const double eps = D.ctl->eps;
  // xdefer: x += alpha d' is left to the next K1 (which streams d anyway); only an x parked in t
  // by a fresh-residual K1 is moved back here
  const bool xd = D.xdefer != 0;
  const bool xint = xd && (D.st[sys].flags & FL_XINT) != 0;
  const double* dn = par ? D.d0 : D.d1;
  const double* rc = par ? D.r1 : D.r0;
  double* rn = par ? D.r0 : D.r1;
  double* gr = reinterpret_cast<double*>(smraw);  // [ND][GR]
  double* rp = gr + ND * GR;                        // [GR]  r (bulk copy) -> r' in place
  double* tr = rp + GR;                             // [TR]
  double* qs = tr + TR;                             // [P][C]
  unsigned char* mk = reinterpret_cast<unsigned char*>(qs + P * C);  // [GR]
  // Ranges alternate direction inside a system: even ranges stream upwards, odd ones downwards,
  // so two neighbouring ranges reach their shared boundary -- and read the 2*NH-chunk halo each
  // needs from the other side -- at the same time (both at their ends or both at their starts):
  // the second read is an L2 hit instead of an HBM re-read.  Rings are indexed by ROW (chunk
  // c_rel = k upwards, K - 1 - k downwards, relative to LB), so neighbour arithmetic and every
  // row's summation order are the same in both directions.
  // LB / the top are 16-row aligned so every bulk copy is 16-byte aligned.
  const bool down = ((b - D.sys_rng0[sys]) & 1) != 0;
  const long long R0a = R0 & ~15LL, R1a = (R1 + 15) & ~15LL;
  const int K = (int)(((down ? R1a - R0 : R1 - R0a) + C - 1) / C) + 4 * NH;  // output chunks + warm-up + lead-out
  const long long LB = down ? R1a + 2LL * NH * C - (long long)K * C : R0a - 2LL * NH * C;
  auto crel = [&](int k) { return down ? K - 1 - k : k; };
  auto rel = [&](long long v) { return (int)(v - LB < -1 ? -1 : (v - LB > (1LL << 30) ? (1LL << 30) : v - LB)); };
  const int s0r = rel(s0), s1r = rel(s1), R0r = rel(R0), R1r = rel(R1);
  const Own ow = own_get<PART>(D, sys);
  const int o0r = PART ? rel(ow.o0) : INT_MIN, o1r = PART ? rel(ow.o1) : INT_MAX;
  int off[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) off[d] = D.dia.off[d];
  auto issue = [&](int k) {
    const int cr = crel(k);
    const int ss = k % P, gs = (cr % NG) * C;
    const long long row = LB + (long long)cr * C;
    mbar_arrive_expect_tx(&bars[ss], (uint32_t)((2 + ND) * C * 8 + C));
    bulk_g2s(rp + gs, rc + row, C * 8, &bars[ss]);
    bulk_g2s(qs + ss * C, D.q + row, C * 8, &bars[ss]);
#pragma unroll
    for (int d = 0; d < ND; ++d) bulk_g2s(gr + d * GR + gs, D.dia.gv[d] + row, C * 8, &bars[ss]);
    bulk_g2s(mk + gs, D.dia.mask + row, C, &bars[ss]);
  };
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < P; ++q) {
      mbar_init(&bars[q], 1);
      mbar_init(&empty[q], PR / 32);
    }
    mbar_init_fence();
  }
  __syncthreads();
  double prr = 0.0, prs = 0.0;
  if (tid >= PR) {  // producer warp: chunk c once step c - P (the last user of its slots) is done
    if (tid == PR)
      for (int c = 0; c < K; ++c) {
        if (c >= P) mbar_wait(&empty[c % P], (uint32_t)((c / P - 1) & 1));
        issue(c);
      }
  } else
  for (int k = 0; k < K; ++k) {
    // x, d of this step's output chunk: plain loads, in flight across the wait and phases A, B
    const int mm = k - 2 * NH;
    const int cm = crel(mm);
    const int li = cm * C + tid;
    const bool own_c = mm >= 2 * NH && li >= R0r && li < R1r;
    double xo = 0.0, dd = 0.0;
    if (own_c && !xd) {
      xo = D.x[LB + li];
      dd = __ldg(dn + LB + li);
    } else if (own_c && xint) {
      xo = D.t[LB + li];
    }
    mbar_wait(&bars[k % P], (uint32_t)((k / P) & 1));
    {  // A: r' of the lead chunk, in place over its r
      const int ck = crel(k);
      const int lj = ck * C + tid, ix = (ck % NG) * C + tid;
      double v = sub(rp[ix], mul(alpha, qs[(k % P) * C + tid]));
      v = (lj >= s0r && lj < s1r) ? v : 0.0;
      if (lj >= R0r && lj < R1r) {
        rn[LB + lj] = v;
        if (lj >= o0r && lj < o1r) prr += mul(v, v);
      }
      rp[ix] = v;
    }
    named_bar_sync(1, PR);
    const int u = k - NH;
    if (u >= NH) {  // B: t of chunk u (add.at order over G's mirror diagonals)
      const int cu = crel(u);
      const int lj = cu * C + tid, base = (cu % NG) * C + tid;
      const unsigned int m = mk[base];
      double p[ND];
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        const int ix = ring_nb<ND>(base, off, d, GR);
        p[d] = mul(gr[(ND - 1 - d) * GR + ix], rp[ix]);
      }
      const double v = combine_seq<ND>(p, m);
      tr[(cu % NT) * C + tid] = (lj >= s0r && lj < s1r) ? v : 0.0;
    }
    named_bar_sync(1, PR);
    if (own_c) {  // C: s and x of chunk mm (s of owned rows only: ghost s comes from the neighbours)
      const long long i = LB + li;
      if (!xd) D.x[i] = add(xo, mul(alpha, dd));
      else if (xint) D.x[i] = xo;
      if (li >= o0r && li < o1r) {
        const int io = (cm % NG) * C + tid, tb = (cm % NT) * C + tid;
        const unsigned int m = mk[io];
        double p[ND];
#pragma unroll
        for (int d = 0; d < ND; ++d) p[d] = mul(gr[d * GR + io], tr[ring_nb<ND>(tb, off, d, TR)]);
        const double y = combine_numpy<ND>(p, m);
        const double rni = rp[io];
        const double si = add(y, mul(eps, rni));
        store_s(D, ow, i, si);
        prs += mul(rni, si);
      }
    }
    // step k done: its lead chunk's staging and the ring slot read last by phase C are free
    // (the next phase A of this thread follows a named barrier with every other consumer)
    if ((tid & 31) == 0) mbar_arrive(&empty[k % P]);
  }
  if (arrive(D, D.sys_rng0, sys, prr, prs, red, &flag)) {
    double rr, rs;
    gather_partials2(D, D.sys_rng0, sys, rr, rs);
    if (threadIdx.x == 0) {
      if (PART) {
        part_fin(D, sys, FIN_K23, rr, rs, 0);
      } else {
        D.st[sys].rr = rr;
        if (xd) D.st[sys].flags = (D.st[sys].flags & ~(FL_XINT | FL_DPAR)) | FL_XPEND | (par ? FL_DPAR : 0);
        fin_k3(D, sys, rs, 0);
      }
    }
  }
}

// ------------------------------------------------------------------ sliding-window K1
// K1 as a stream over the same ranges: per step the bulk-copy engine brings the lead chunk's
// s, d, A diagonals (the lower half only when A is stored by it) and mask; then
//   A  d' = s + beta d              lead chunk k   -> d' ring (own rows: d' to HBM)
//   Q  q  = A d'                    chunk k - NH   (numpy order; partial d'.q)
// One CTA barrier per step.  A pending fresh-residual check (rare: only after a candidate
// convergence) runs after the stream over the range's own rows with direct loads.
// CS (coefficient stencil, 5-point gen_poisson2d matrices): the ring holds the node
// coefficients instead of A's diagonals (8 instead of 24 B/row) and A's entries are recomputed
// bitwise (stencil5); the +-W neighbours of chunk u reach back to chunk u - NH, so the ring
// spans u - NH .. k + P - 1.
#ifndef SG_SWP_CS
#define SG_SWP_CS 6
#endif
template <int FMT, int ND, int NH, bool CS = false>
struct Sw1 {
  static constexpr int C = kSwC;
  // chunks in flight (incl. the current one); the coefficient ring's smaller footprint buys depth
  static constexpr int P = CS ? SG_SWP_CS : 4;
  static constexpr int NA = CS ? 1 : (FMT == 2 ? ND / 2 + 1 : ND);  // diagonals (or coefficients) streamed
  static constexpr bool BOTHDIR = true;  // the ring holds the row-chunks on both sides of u
  // A / mask ring chunks u - NH .. k + P - 1 (the rows behind chunk u: the stencil's +-W
  // neighbours, the lower-half A's upper entries when streaming downwards)
  static constexpr int NR = P + 2 * NH;
  static constexpr int RING = NR * C;
  static constexpr int DRING = pow2ceil((2 * NH + 2) * C); // d' ring: chunks u - NH .. k + 1
  static constexpr int DM = DRING - 1;
  // bytes: A [NA][RING] | d' [DRING] | staging [P][2][C] (s, d) | mask [RING]
  static constexpr size_t SMEM = (size_t)NA * RING * 8 + (size_t)DRING * 8 + (size_t)P * 2 * C * 8 + RING;
};

template <int FMT, int ND, int NH, bool CS = false, bool PART = false>
__global__ void __launch_bounds__(PR, 5) k_iter1_sw(Dev D, int par) {
  static_assert(!CS || (FMT == 2 && ND == 5), "coefficient stencil: 5-point symmetric DIA only");
  using G = Sw1<FMT, ND, NH, CS>;
  constexpr int C = G::C, P = G::P, NA = G::NA, NR = G::NR, RING = G::RING, DM = G::DM;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bars[P];
  __shared__ double red[PR / 32];
  __shared__ int flag;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int sys = D.rng_sys[b];
  const int status = D.st[sys].status;
  if (status == ST_DONE) return;
  long long s0, s1;
  sys_bounds(D, sys, s0, s1);
  const long long R0 = D.rng_r0[b];
  const long long R1 = R0 + D.rng_len < s1 ? R0 + D.rng_len : s1;
  const bool run = status == ST_RUN;
  const int flags = D.st[sys].flags;
  const bool fresh = run ? (flags & FL_FRESH) != 0 : true;
  // deferred x update of the previous fused K2+K3: x += alpha_prev d (d = this kernel's d_old).
  // In place while streaming; when a fresh residual is due, other CTAs read neighbours' x in this
  // kernel, so the updated x goes to t instead and b - A x reads x + alpha d on the fly.
  const bool pend = D.xdefer && (flags & FL_XPEND) != 0;
  const double alpha_p = D.st[sys].alpha;
  const double beta = D.st[sys].beta;
  const double* dc = par ? D.d1 : D.d0;
  double* dn = par ? D.d0 : D.d1;
  double* rc = par ? D.r1 : D.r0;
  const Own ow = own_get<PART>(D, sys);
  double pdq = 0.0, prr = 0.0;
  if (run) {
    double* ar = reinterpret_cast<double*>(smraw);  // [NA][RING]
    double* dp = ar + NA * RING;                      // [DRING]
    double* stg = dp + G::DRING;                      // [P][2][C]
    unsigned char* mk = reinterpret_cast<unsigned char*>(stg + P * 2 * C);
    // alternating stream direction per range, row-indexed rings (see k_iter23_sw)
    const bool down = G::BOTHDIR && ((b - D.sys_rng0[sys]) & 1) != 0;
    const long long R0a = R0 & ~15LL, R1a = (R1 + 15) & ~15LL;
    const int K = (int)(((down ? R1a - R0 : R1 - R0a) + C - 1) / C) + 2 * NH;
    const long long LB = down ? R1a + (long long)NH * C - (long long)K * C : R0a - (long long)NH * C;
    auto crel = [&](int k) { return down ? K - 1 - k : k; };
    auto rel = [&](long long v) { return (int)(v - LB < -1 ? -1 : (v - LB > (1LL << 30) ? (1LL << 30) : v - LB)); };
    const int s0r = rel(s0), s1r = rel(s1), R0r = rel(R0), R1r = rel(R1);
    const int o0r = PART ? rel(ow.o0) : INT_MIN, o1r = PART ? rel(ow.o1) : INT_MAX;
    int off[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) off[d] = D.dia.off[d];
    auto issue = [&](int k) {
      const int cr = crel(k);
      const int ss = k % P, gs = (cr % NR) * C;
      double* st = stg + ss * 2 * C;
      const long long row = LB + (long long)cr * C;
      mbar_arrive_expect_tx(&bars[ss], (uint32_t)((2 + NA) * C * 8 + C));
      bulk_g2s(st, D.s + row, C * 8, &bars[ss]);
      bulk_g2s(st + C, dc + row, C * 8, &bars[ss]);
      if (CS) bulk_g2s(ar + gs, D.coef + row, C * 8, &bars[ss]);
      else {
#pragma unroll
        for (int d = 0; d < NA; ++d) bulk_g2s(ar + d * RING + gs, D.dia.av[d] + row, C * 8, &bars[ss]);
      }
      bulk_g2s(mk + gs, D.dia.mask + row, C, &bars[ss]);
    };
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < P; ++q) mbar_init(&bars[q], 1);
      mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0)
      for (int k = 0; k < P - 1 && k < K; ++k) issue(k);
    const bool xupd = pend && !fresh;
    double xo_n = 0.0;  // x of the lead chunk's own rows, loaded one step ahead
    if (xupd && crel(0) * C + tid >= R0r && crel(0) * C + tid < R1r) xo_n = D.x[LB + crel(0) * C + tid];
    int ks = 0;        // k % P, kept incrementally (no division per step)
    uint32_t kph = 0;  // (k / P) & 1
    for (int k = 0; k < K; ++k) {
      const double* st = stg + ks * 2 * C;
      const int lj = crel(k) * C + tid;
      bool xown = false;
      double xo = 0.0;
      if (xupd) {  // uniform: off unless the x update is deferred into K1 (SG_PCG_XDEFER)
        xown = lj >= R0r && lj < R1r;
        xo = xo_n;
        const int ljn = crel(k + 1) * C + tid;  // the next lead chunk's row (either direction)
        if (k + 1 < K && ljn >= R0r && ljn < R1r) xo_n = D.x[LB + ljn];
      }
      mbar_wait(&bars[ks], kph);
      {  // d' of the lead chunk (and the deferred x update of its own rows)
        double v = add(st[tid], mul(beta, st[C + tid]));
        v = (lj >= s0r && lj < s1r) ? v : 0.0;
        if (lj >= R0r && lj < R1r) dn[LB + lj] = v;
        if (xown) D.x[LB + lj] = add(xo, mul(alpha_p, st[C + tid]));
        dp[lj & DM] = v;
      }
      __syncthreads();
      if (tid == 0 && k + P - 1 < K) issue(k + P - 1);
      const int u = k - NH;
      if (u >= 0) {  // q of chunk u
        const int cu = crel(u);
        const int li = cu * C + tid;
        if (li >= R0r && li < R1r) {
          const int io = (cu % NR) * C + tid;
          const unsigned int m = mk[io];
          double p[ND];
          if constexpr (CS) {
            double a[5];
            // a power-of-two ring (the coefficient ring: P + 2 NH chunks) wraps with one mask
            auto nb = [&](int d) {
              if constexpr ((RING & (RING - 1)) == 0) return (io + off[d]) & (RING - 1);
              else return ring_nb<ND>(io, off, d, RING);
            };
            stencil5(ar[io], ar[nb(0)], ar[nb(1)], ar[nb(3)], ar[nb(4)], m, D.ihx2, D.ihy2, a);
#pragma unroll
            for (int d = 0; d < ND; ++d) p[d] = mul(a[d], dp[(li + off[d]) & DM]);
          } else {
#pragma unroll
            for (int d = 0; d < ND; ++d) {
              const int ix = ring_nb<ND>(io, off, d, RING);
              // FMT 2: an upper entry (i, i+off) is the lower mirror entry at row i+off
              const double a = (FMT == 2 && d > ND / 2) ? ar[(ND - 1 - d) * RING + ix] : ar[d * RING + io];
              p[d] = mul(a, dp[(li + off[d]) & DM]);
            }
          }
          const double qi = combine_numpy<ND>(p, m);
          D.q[LB + li] = qi;
          if (li >= o0r && li < o1r) pdq += mul(dp[li & DM], qi);
        }
      }
      if (++ks == P) {
        ks = 0;
        kph ^= 1u;
      }
    }
  }
  if (fresh) {  // r_fresh = b - A x over the range's own rows (direct loads)
    for (long long i = R0 + tid; i < R1; i += PR) {
      const unsigned int m = D.dia.mask[i];
      double ax;
      if (pend) {  // x + alpha_prev d, exactly the deferred update; the updated x goes to t
        const XF xf{D.x, dc, alpha_p};
        ax = FMT == 2 ? dia_row_numpy_sym<ND, 1>(D.dia, D.dia.av, (int)i, m, xf)
                      : dia_row_numpy<ND, 1>(D.dia, D.dia.av, (int)i, m, xf);
        D.t[i] = add(D.x[i], mul(alpha_p, dc[i]));
      } else {
        ax = FMT == 2 ? dia_row_numpy_sym<ND, 0>(D.dia, D.dia.av, (int)i, m, XF{D.x, nullptr, 0.0})
                      : dia_row_numpy<ND, 0>(D.dia, D.dia.av, (int)i, m, XF{D.x, nullptr, 0.0});
      }
      const double rf = sub(D.b[i], ax);
      if (run) rc[i] = rf;
      if (owned(ow, i)) prr += mul(rf, rf);
    }
  }
  if (arrive(D, D.sys_rng0, sys, pdq, prr, red, &flag)) {
    double dq, rrf;
    gather_partials2(D, D.sys_rng0, sys, dq, rrf);
    if (threadIdx.x == 0) {
      if (PART) {
        part_fin(D, sys, FIN_K1, dq, rrf, run);
      } else {
        if (pend) D.st[sys].flags = (D.st[sys].flags & ~(FL_XPEND | FL_DPAR)) | (fresh ? FL_XINT : 0);
        fin_k1(D, sys, run, dq, rrf);
      }
    }
  }
}

// ------------------------------------------------------------------ 2-D strip sliding window
// Wide 5-point grids (offsets {-W, -1, 0, 1, W}, W > 512: the north-star 2048^2 shape) do not
// fit a 1-D halo ring, so the stream runs over grid LINES inside a column STRIP instead: a CTA
// owns columns [x0, x0 + 256) of lines [y0, y1) of one system and walks them line by line.  A
// line segment is loaded with E = 2 columns of x-halo on each side (positions p = x - x0 + 2,
// 0 <= p < SP); the +-W neighbours are the adjacent line slots of the ring and the +-1
// neighbours are p +- 1, so all of it is plain 1-D DIA arithmetic (a position past the strip
// edge is simply the neighbouring row).  Same phases, roundings and summation orders as the
// 1-D kernels; only the partial sums are grouped per (strip, line range).
#ifndef SG_STRIP_C
#define SG_STRIP_C 256
#endif
constexpr int kStripC = SG_STRIP_C;        // columns per strip (one per thread of the CTA)
constexpr int kStripE = 2;                 // x-halo columns on each side
constexpr int kStripSP = kStripC + 2 * kStripE;  // 260 positions per line segment (2080 B)
constexpr int kStripMK = kStripSP + 28;    // mask window: 16-row aligned start, 288 bytes
constexpr int kStripRL = 4;                // ring lines (power of two)

// (line, column) displacement of the 5-point diagonals d = 0..4 (offsets -W, -1, 0, 1, W)
__device__ __forceinline__ constexpr int s5a(int d) { return d == 0 ? -1 : (d == 4 ? 1 : 0); }
__device__ __forceinline__ constexpr int s5b(int d) { return d == 1 ? -1 : (d == 3 ? 1 : 0); }

// G of a wide grid in strip blocks: block (strip sx, extended line) = G's five diagonals at the
// SP positions of that line segment ([5][SP] doubles) followed by their mask bytes.  Extended lines
// are laid out per strip over all systems, each system framed by two zero lines on each side
// (the warm-up / lead-out lines of its first and last ranges); positions outside the system are
// zero (their products are masked out by the centre rows' masks).  Built once per solve after G's
// diagonals, so the strip K2+K3 streams one contiguous ~10 KB copy per line instead of six ~2 KB
// ones -- small bulk copies cap the copy engine's bandwidth (profiles/r03_stream_bw.txt), while
// r, q, x, d come by plain coalesced loads issued a step ahead.
constexpr int kStripMKB = (kStripSP + 15) / 16 * 16;
constexpr int kStripBB = 5 * kStripSP * 8 + kStripMKB;  // bytes per block (16-byte multiple)

__global__ void k_strip_gblocks(Dev D, unsigned char* blk) {
  const int sys = blockIdx.y;
  long long s0, s1;
  sys_bounds(D, sys, s0, s1);
  const long long W = D.dia.W, nl = (s1 - s0) / W, L = D.gblk_L;
  const long long ns = (W + kStripC - 1) / kStripC;
  const long long gl0 = s0 / W + 4LL * sys;
  const long long tot = ns * (nl + 4) * kStripSP;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(e % kStripSP);
    const long long t = e / kStripSP;
    const long long yl = t % (nl + 4), sx = t / (nl + 4);
    const long long row = s0 + (yl - 2) * W + sx * kStripC - kStripE + p;
    const bool in = yl >= 2 && yl < nl + 2 && row >= s0 && row < s1;
    unsigned char* bp = blk + (sx * L + gl0 + yl) * kStripBB;
    double* g = reinterpret_cast<double*>(bp);
#pragma unroll
    for (int d = 0; d < 5; ++d) g[d * kStripSP + p] = in ? D.dia.gv[d][row] : 0.0;
    bp[5 * kStripSP * 8 + p] = in ? D.dia.mask[row] : (unsigned char)0;
  }
}

#ifndef SG_STRIP_PG
#define SG_STRIP_PG 2
#endif

struct Strip23 {
  static constexpr int P = SG_STRIP_PG;  // G blocks in flight (incl. the current line)
  static constexpr int RG = P + 2;       // G block ring (lines k - 2 .. k + P - 1)
  // bytes: G blocks [RG][BB] | r' [RL][SP] | t [RL][SP]
  static constexpr size_t SMEM = (size_t)RG * kStripBB + (size_t)2 * kStripRL * kStripSP * 8;
};

// Position-relative bounds: row j = rb + p of a line segment lies in [lo, hi) iff p lies in
// [prel(lo - rb), prel(hi - rb)) -- per-line (uniform) 64-bit work, per-position 32-bit compares.
__device__ __forceinline__ int prel(long long v) { return (int)(v < -1 ? -1 : (v > (1 << 20) ? (1 << 20) : v)); }

template <bool PART = false>
__global__ void __launch_bounds__(kStripC, PART ? 3 : 768 / kStripC) k_iter23_s5(Dev D, int par) {
  constexpr int SP = kStripSP, RL = kStripRL, P = Strip23::P, RG = Strip23::RG, C = kStripC, E = kStripE;
  constexpr int BBD = kStripBB / 8, MKO = 5 * SP * 8;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bars[P];
  __shared__ double red[kStripC / 32];
  __shared__ int flag;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int sys = D.rng_sys[b];
  trace_stamp(D, 1, 0);
  if (D.st[sys].status != ST_RUN) return;
  long long s0, s1;
  sys_bounds(D, sys, s0, s1);
  const long long W = D.dia.W;
  const long long r0 = D.rng_r0[b] - s0;
  const int x0 = (int)(r0 % W);
  const long long y0 = r0 / W, nl = (s1 - s0) / W;
  const long long y1 = y0 + D.rng_len < nl ? y0 + D.rng_len : nl;
  const int cx = (int)(W - x0 < C ? W - x0 : C);  // own columns of this strip
  const Own ow = own_get<PART>(D, sys);
  const double alpha = D.st[sys].alpha;
  const double eps = D.ctl->eps;
  const double* dn = par ? D.d0 : D.d1;
  const double* rc = par ? D.r1 : D.r0;
  double* rn = par ? D.r0 : D.r1;
  double* gb = reinterpret_cast<double*>(smraw);  // [RG][BBD]
  double* rp = gb + RG * BBD;                       // [RL][SP]
  double* tr = rp + RL * SP;                        // [RL][SP]
  const int K = (int)(y1 - y0) + 4;
  // row of position 0 of step k's lead line (line y0 - 2 + k)
  const long long rb0 = s0 + (y0 - 2) * W + x0 - E;
  // the block of step k's line (extended line y0 + k of this system)
  const unsigned char* gsrc = D.gblk + ((long long)(x0 / C) * D.gblk_L + s0 / W + 4LL * sys + y0) * kStripBB;
  auto gline = [&](int k) { return gb + (k % RG) * BBD; };
  auto issue = [&](int k) {
    mbar_arrive_expect_tx(&bars[k % P], (uint32_t)kStripBB);
    bulk_g2s(gline(k), gsrc + (long long)k * kStripBB, kStripBB, &bars[k % P]);
  };
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < P; ++q) mbar_init(&bars[q], 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0)
    for (int k = 0; k < P - 1 && k < K; ++k) issue(k);
  // r, q of the lead line segment: plain loads one step ahead (guard bands cover the lines
  // beyond the system; those values are masked to zero)
  const bool two = tid + C < SP;  // this thread also holds halo position tid + C
  double nr[2] = {0.0, 0.0}, nq[2] = {0.0, 0.0};
  auto load_rq = [&](long long rb) {
    nr[0] = __ldcs(rc + rb + tid);
    nq[0] = __ldcs(D.q + rb + tid);
    if (two) {
      nr[1] = __ldcs(rc + rb + tid + C);
      nq[1] = __ldcs(D.q + rb + tid + C);
    }
  };
  load_rq(rb0);
  double prr = 0.0, prs = 0.0;
  for (int k = 0; k < K; ++k) {
    const double cr[2] = {nr[0], nr[1]}, cq[2] = {nq[0], nq[1]};
    const long long rb = rb0 + (long long)k * W;  // lead line (A)
    if (k + 1 < K) load_rq(rb + W);
    // x, d of this step's output line (phase C): in flight across phases A and B
    const int mm = k - 2;
    const long long rbm = rb - 2 * W;
    const bool ownc = mm >= 2 && tid < cx && mm - 2 < y1 - y0;
    double xo = 0.0, dd = 0.0;
    if (ownc) {
      xo = D.x[rbm + E + tid];
      dd = __ldcs(dn + rbm + E + tid);
    }
    {  // A: r' of the lead line segment
      const int lo = prel(s0 - rb), hi = prel(s1 - rb);
      const bool lown = k >= 2 && k - 2 < y1 - y0;  // the lead line is one of the range's own lines
      const int olo = PART ? prel(ow.o0 - rb) : INT_MIN, ohi = PART ? prel(ow.o1 - rb) : INT_MAX;
      const int ls = k & (RL - 1);
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int p = tid + h2 * C;
        if (h2 == 0 || two) {
          double v = sub(cr[h2], mul(alpha, cq[h2]));
          v = (p >= lo && p < hi) ? v : 0.0;
          if (lown && p >= E && p < E + cx) {
            rn[rb + p] = v;
            if (p >= olo && p < ohi) prr += mul(v, v);
          }
          rp[ls * SP + p] = v;
        }
      }
    }
    mbar_wait(&bars[k % P], (uint32_t)((k / P) & 1));  // G of line k (B's u + 1 neighbour)
    __syncthreads();
    if (tid == 0 && k + P - 1 < K) issue(k + P - 1);
    const int u = k - 1;
    if (u >= 1) {  // B: t on positions 1 .. SP-2 of line u (add.at order over G's mirrors)
      const long long rbu = rb - W;
      const int lo = prel(s0 - rbu), hi = prel(s1 - rbu);
      const unsigned char* mu = reinterpret_cast<const unsigned char*>(gline(u)) + MKO;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int p = 1 + tid + h2 * C;
        if (h2 == 0 || p < SP - 1) {
          const unsigned int m = mu[p];
          double pr[5];
#pragma unroll
          for (int d = 0; d < 5; ++d)
            pr[d] = mul(gline(u + s5a(d))[(4 - d) * SP + p + s5b(d)],
                        rp[((u + s5a(d)) & (RL - 1)) * SP + p + s5b(d)]);
          const double v = combine_seq<5>(pr, m);
          tr[(u & (RL - 1)) * SP + p] = (p >= lo && p < hi) ? v : 0.0;
        }
      }
    }
    __syncthreads();
    if (ownc) {  // C: own columns of line mm
      const int p = tid + E;
      const long long i = rbm + p;
      D.x[i] = add(xo, mul(alpha, dd));
      if (owned(ow, i)) {  // s of owned rows only: ghost s comes from the neighbour partitions
        const int ls = mm & (RL - 1);
        const double* gm = gline(mm);
        const unsigned int m = reinterpret_cast<const unsigned char*>(gm)[MKO + p];
        double pr[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) pr[d] = mul(gm[d * SP + p], tr[((mm + s5a(d)) & (RL - 1)) * SP + p + s5b(d)]);
        const double y = combine_numpy<5>(pr, m);
        const double rni = rp[ls * SP + p];
        const double si = add(y, mul(eps, rni));
        store_s(D, ow, i, si);
        prs += mul(rni, si);
      }
    }
  }
  trace_stamp(D, 1, 1);
  const bool last = arrive(D, D.sys_rng0, sys, prr, prs, red, &flag);
  trace_stamp(D, 1, 2);
  if (last) {
    double rr, rs;
    gather_partials2(D, D.sys_rng0, sys, rr, rs);
    if (threadIdx.x == 0) {
      if (PART) {
        part_fin(D, sys, FIN_K23, rr, rs, 0);
      } else {
        D.st[sys].rr = rr;
        fin_k3(D, sys, rs, 0);
      }
    }
    trace_stamp(D, 1, 3);
  }
}

// K1 on strips: d' = s + beta d over each lead line segment, q = A d' on the own columns.
// CS (coefficient stencil, gen_poisson2d matrices; see k_iter1_sw): the A ring holds one node
// coefficient per position instead of A's three lower diagonals and the row's five entries are
// recomputed bitwise; the south neighbour's coefficient (line u - 1) makes that ring RA = 8 lines.
template <int FMT, bool CS = false>
struct Strip1 {
  static constexpr int P = 3;
  static constexpr int NA = CS ? 1 : (FMT == 2 ? 3 : 5);
  static constexpr int RA = CS ? 8 : kStripRL;  // A / coefficient ring lines (power of two)
  // bytes: A [NA][RA][SP] | d' [RL][SP] | staging [P][2][SP] (s, d) | mask [RL][MK]
  static constexpr size_t SMEM = (size_t)NA * RA * kStripSP * 8 + (size_t)kStripRL * kStripSP * 8 +
                                 (size_t)P * 2 * kStripSP * 8 + (size_t)kStripRL * kStripMK;
};

template <int FMT, bool PART = false, bool CS = false>
__global__ void __launch_bounds__(kStripC, 1024 / kStripC) k_iter1_s5(Dev D, int par) {
  static_assert(!CS || (FMT == 2 && !PART), "coefficient stencil: symmetric 5-point DIA, one partition");
  using G = Strip1<FMT, CS>;
  constexpr int SP = kStripSP, RL = kStripRL, P = G::P, NA = G::NA, RA = G::RA, E = kStripE;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bars[P];
  __shared__ double red[kStripC / 32];
  __shared__ int flag;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int sys = D.rng_sys[b];
  const int status = D.st[sys].status;
  if (status == ST_DONE) return;
  long long s0, s1;
  sys_bounds(D, sys, s0, s1);
  const long long W = D.dia.W;
  const long long r0 = D.rng_r0[b] - s0;
  const int x0 = (int)(r0 % W);
  const long long y0 = r0 / W, nl = (s1 - s0) / W;
  const long long y1 = y0 + D.rng_len < nl ? y0 + D.rng_len : nl;
  const int cx = (int)(W - x0 < kStripC ? W - x0 : kStripC);
  const Own ow = own_get<PART>(D, sys);
  const bool run = status == ST_RUN;
  const bool fresh = run ? (D.st[sys].flags & FL_FRESH) != 0 : true;
  const double beta = D.st[sys].beta;
  const double* dc = par ? D.d1 : D.d0;
  double* dn = par ? D.d0 : D.d1;
  double* rc = par ? D.r1 : D.r0;
  auto rowof = [&](long long line, int p) { return s0 + line * W + x0 - E + p; };
  double pdq = 0.0, prr = 0.0;
  if (run) {
    double* ar = reinterpret_cast<double*>(smraw);  // [NA][RA][SP]
    double* dp = ar + NA * RA * SP;                   // [RL][SP]
    double* stg = dp + RL * SP;                       // [P][2][SP]
    unsigned char* mk = reinterpret_cast<unsigned char*>(stg + P * 2 * SP);
    const long long LBl = y0 - 1;
    const int K = (int)(y1 - y0) + 2;
    auto issue = [&](int k) {
      const int ss = k % P, ls = k & (RL - 1), la = k & (RA - 1);
      const long long row = rowof(LBl + k, 0);
      mbar_arrive_expect_tx(&bars[ss], (uint32_t)((2 + NA) * SP * 8 + kStripMK));
      bulk_g2s(stg + ss * 2 * SP, D.s + row, SP * 8, &bars[ss]);
      bulk_g2s(stg + ss * 2 * SP + SP, dc + row, SP * 8, &bars[ss]);
      if (CS) bulk_g2s(ar + la * SP, D.coef + row, SP * 8, &bars[ss]);
      else {
#pragma unroll
        for (int d = 0; d < NA; ++d) bulk_g2s(ar + (d * RA + la) * SP, D.dia.av[d] + row, SP * 8, &bars[ss]);
      }
      bulk_g2s(mk + ls * kStripMK, D.dia.mask + (row - 14), kStripMK, &bars[ss]);
    };
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < P; ++q) mbar_init(&bars[q], 1);
      mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0)
      for (int k = 0; k < P - 1 && k < K; ++k) issue(k);
    for (int k = 0; k < K; ++k) {
      const double* st = stg + (k % P) * 2 * SP;
      mbar_wait(&bars[k % P], (uint32_t)((k / P) & 1));
      {  // d' of the lead line segment
        const long long line = LBl + k;
        const int ls = k & (RL - 1);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int p = tid + h2 * kStripC;
          if (p < SP) {
            const long long j = rowof(line, p);
            double v = add(st[p], mul(beta, st[SP + p]));
            v = (j >= s0 && j < s1) ? v : 0.0;
            const int x = x0 - E + p;
            if (line >= y0 && line < y1 && x >= x0 && x < x0 + cx) dn[j] = v;
            dp[ls * SP + p] = v;
          }
        }
      }
      __syncthreads();
      if (tid == 0 && k + P - 1 < K) issue(k + P - 1);
      const int u = k - 1;
      const long long line = LBl + u;
      if (u >= 1 && tid < cx && line >= y0 && line < y1) {  // q of the own columns of line u
        const int p = tid + E;
        const int ls = u & (RL - 1), la = u & (RA - 1);
        const unsigned int m = mk[ls * kStripMK + p + 14];
        double pr[5];
        if constexpr (CS) {
          const double* cu = ar + la * SP + p;
          double a[5];
          stencil5(cu[0], ar[((u - 1) & (RA - 1)) * SP + p], cu[-1], cu[1], ar[((u + 1) & (RA - 1)) * SP + p], m,
                   D.ihx2, D.ihy2, a);
#pragma unroll
          for (int d = 0; d < 5; ++d) pr[d] = mul(a[d], dp[((u + s5a(d)) & (RL - 1)) * SP + p + s5b(d)]);
        } else {
#pragma unroll
          for (int d = 0; d < 5; ++d) {
            // FMT 2: an upper entry (i, i+off) is the lower mirror entry at row i+off
            double a;
            if (FMT == 2 && d > 2) a = ar[((4 - d) * RA + ((u + s5a(d)) & (RA - 1))) * SP + p + s5b(d)];
            else a = ar[(d * RA + la) * SP + p];
            pr[d] = mul(a, dp[((u + s5a(d)) & (RL - 1)) * SP + p + s5b(d)]);
          }
        }
        const double qi = combine_numpy<5>(pr, m);
        const long long i = rowof(line, p);
        D.q[i] = qi;
        if (owned(ow, i)) pdq += mul(dp[ls * SP + p], qi);
      }
    }
  }
  if (fresh) {  // r_fresh = b - A x over the range's own rows (direct loads)
    for (long long line = y0; line < y1; ++line) {
      if (tid >= cx) break;
      const long long i = s0 + line * W + x0 + tid;
      const unsigned int m = D.dia.mask[i];
      const double ax = FMT == 2 ? dia_row_numpy_sym<5, 0>(D.dia, D.dia.av, (int)i, m, XF{D.x, nullptr, 0.0})
                                 : dia_row_numpy<5, 0>(D.dia, D.dia.av, (int)i, m, XF{D.x, nullptr, 0.0});
      const double rf = sub(D.b[i], ax);
      if (run) rc[i] = rf;
      if (owned(ow, i)) prr += mul(rf, rf);
    }
  }
  if (arrive(D, D.sys_rng0, sys, pdq, prr, red, &flag)) {
    double dq, rrf;
    gather_partials2(D, D.sys_rng0, sys, dq, rrf);
    if (threadIdx.x == 0) { if (PART) part_fin(D, sys, FIN_K1, dq, rrf, run); else fin_k1(D, sys, run, dq, rrf); }
  }
}

// K1 on strips, TWO lines per step (coefficient stencil, the C5 path): per step the bulk-copy
// engine brings a PAIR of lead line segments (s, d, coefficients, mask), d' of both is formed,
// one CTA barrier, then q of the two lines behind them.  Same per-row arithmetic and the same
// per-thread summation order as k_iter1_s5 (bit-identical), half the barriers per row and two
// independent rows per thread between them.  Rings of 8 lines: a step reads d' / coefficients of
// lines 2k-2 .. 2k+1 while the next pair's d' and the copies of pair k+P-1 land elsewhere.
struct Strip1P {
  static constexpr int P = 3;   // line pairs in flight
  static constexpr int RL = 8;  // coefficient, d' and mask rings (lines; power of two)
  // bytes: coefficients [RL][SP] | d' [RL][SP] | staging [P][2 lines][s, d][SP] | mask [RL][MK]
  static constexpr size_t SMEM = (size_t)2 * RL * kStripSP * 8 + (size_t)P * 4 * kStripSP * 8 +
                                 (size_t)RL * kStripMK;
};

__global__ void __launch_bounds__(kStripC, 3) k_iter1_s5p(Dev D, int par) {
  constexpr int SP = kStripSP, RL = Strip1P::RL, P = Strip1P::P, E = kStripE;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bars[P];
  __shared__ double red[kStripC / 32];
  __shared__ int flag;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int sys = D.rng_sys[b];
  trace_stamp(D, 0, 0);
  const int status = D.st[sys].status;
  if (status == ST_DONE) return;
  long long s0, s1;
  sys_bounds(D, sys, s0, s1);
  const long long W = D.dia.W;
  const long long r0 = D.rng_r0[b] - s0;
  const int x0 = (int)(r0 % W);
  const long long y0 = r0 / W, nl = (s1 - s0) / W;
  const long long y1 = y0 + D.rng_len < nl ? y0 + D.rng_len : nl;
  const int cx = (int)(W - x0 < kStripC ? W - x0 : kStripC);
  const bool run = status == ST_RUN;
  const bool fresh = run ? (D.st[sys].flags & FL_FRESH) != 0 : true;
  const double beta = D.st[sys].beta;
  const double* dc = par ? D.d1 : D.d0;
  double* dn = par ? D.d0 : D.d1;
  double* rc = par ? D.r1 : D.r0;
  auto rowof = [&](long long line, int p) { return s0 + line * W + x0 - E + p; };
  double pdq = 0.0, prr = 0.0;
  if (run) {
    double* ar = reinterpret_cast<double*>(smraw);  // [RL][SP]
    double* dp = ar + RL * SP;                        // [RL][SP]
    double* stg = dp + RL * SP;                       // [P][2][2][SP]
    unsigned char* mk = reinterpret_cast<unsigned char*>(stg + P * 4 * SP);
    const long long LBl = y0 - 1;
    const int K = (int)(y1 - y0) + 2;  // lines y0 - 1 .. y1
    const int NS = (K + 1) / 2;        // steps
    auto issue = [&](int k) {
      const int ss = k % P;
      const int nlines = 2 * k + 1 < K ? 2 : 1;
      mbar_arrive_expect_tx(&bars[ss], (uint32_t)(nlines * (3 * SP * 8 + kStripMK)));
      for (int h = 0; h < nlines; ++h) {
        const int l = 2 * k + h, lr = l & (RL - 1);
        const long long row = rowof(LBl + l, 0);
        double* st = stg + (ss * 2 + h) * 2 * SP;
        bulk_g2s(st, D.s + row, SP * 8, &bars[ss]);
        bulk_g2s(st + SP, dc + row, SP * 8, &bars[ss]);
        bulk_g2s(ar + lr * SP, D.coef + row, SP * 8, &bars[ss]);
        bulk_g2s(mk + lr * kStripMK, D.dia.mask + (row - 14), kStripMK, &bars[ss]);
      }
    };
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < P; ++q) mbar_init(&bars[q], 1);
      mbar_init_fence();
    }
    __syncthreads();
    if (tid == 0)
      for (int k = 0; k < P - 1 && k < NS; ++k) issue(k);
    for (int k = 0; k < NS; ++k) {
      mbar_wait(&bars[k % P], (uint32_t)((k / P) & 1));
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // d' of lead lines 2k, 2k + 1
        const int l = 2 * k + h;
        if (l < K) {
          const long long line = LBl + l;
          const int lr = l & (RL - 1);
          const double* st = stg + ((k % P) * 2 + h) * 2 * SP;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int p = tid + h2 * kStripC;
            if (p < SP) {
              const long long j = rowof(line, p);
              double v = add(st[p], mul(beta, st[SP + p]));
              v = (j >= s0 && j < s1) ? v : 0.0;
              const int x = x0 - E + p;
              if (line >= y0 && line < y1 && x >= x0 && x < x0 + cx) dn[j] = v;
              dp[lr * SP + p] = v;
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0 && k + P - 1 < NS) issue(k + P - 1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // q of the own columns of lines 2k - 1, 2k
        const int u = 2 * k - 1 + h;
        const long long line = LBl + u;
        if (u >= 1 && tid < cx && line >= y0 && line < y1) {
          const int p = tid + E;
          const int lr = u & (RL - 1);
          const unsigned int m = mk[lr * kStripMK + p + 14];
          const double* cu = ar + lr * SP + p;
          double a[5], pr[5];
          stencil5(cu[0], ar[((u - 1) & (RL - 1)) * SP + p], cu[-1], cu[1], ar[((u + 1) & (RL - 1)) * SP + p], m,
                   D.ihx2, D.ihy2, a);
#pragma unroll
          for (int d = 0; d < 5; ++d) pr[d] = mul(a[d], dp[((u + s5a(d)) & (RL - 1)) * SP + p + s5b(d)]);
          const double qi = combine_numpy<5>(pr, m);
          D.q[rowof(line, p)] = qi;
          pdq += mul(dp[lr * SP + p], qi);
        }
      }
    }
  }
  trace_stamp(D, 0, 1);
  if (fresh) {  // r_fresh = b - A x over the range's own rows (direct loads)
    for (long long line = y0; line < y1; ++line) {
      if (tid >= cx) break;
      const long long i = s0 + line * W + x0 + tid;
      const unsigned int m = D.dia.mask[i];
      const double ax = dia_row_numpy_sym<5, 0>(D.dia, D.dia.av, (int)i, m, XF{D.x, nullptr, 0.0});
      const double rf = sub(D.b[i], ax);
      if (run) rc[i] = rf;
      prr += mul(rf, rf);
    }
  }
  const bool last = arrive(D, D.sys_rng0, sys, pdq, prr, red, &flag);
  trace_stamp(D, 0, 2);
  if (last) {
    double dq, rrf;
    gather_partials2(D, D.sys_rng0, sys, dq, rrf);
    if (threadIdx.x == 0) fin_k1(D, sys, run, dq, rrf);
    trace_stamp(D, 0, 3);
  }
}

}  // namespace sg

using namespace sg;

// ------------------------------------------------------------------ host runtime
struct sg_pcg {
  int S = 0;
  int64_t n = 0;
  int nblk = 0;
  int pre = 0;
  double eps = 0.0;
  std::vector<int64_t> sys_start;
  // device allocations
  void* mem = nullptr;
  Dev D{};
  SysState* st = nullptr;
  Ctl* ctl = nullptr;
  double* hist = nullptr;
  long long hcap = 0;
  unsigned int* pinned_active = nullptr;
  cudaStream_t cap_stream = nullptr;
  std::map<std::vector<int>, cudaGraphExec_t> graphs;
  std::map<std::vector<int>, int> graph_kernels;
  int chunk = 0;
  int64_t period = 0;
  int short_rows = 0;
  int nrng = 0;       // sliding-window ranges
  int num_sms = 148;
  // row partition of one system (sg_pcg_set_partition: group; sg_pcg_set_peers: peer)
  int part = 0;
  void* part_mem = nullptr;   // own / push tables, group sums and counter
  void* red_mem = nullptr;    // peer mode: gsum [2][R][2] + flags [R] + epoch (CUDA IPC exported)
  int red_world = 0;
  int64_t part_n = 0;         // rows of the whole partitioned system (max_iters default 20 n)
  std::vector<void*> peer_maps;  // IPC mappings opened by sg_pcg_set_peers
  int strip = 0;      // wide 5-point grid: 2-D strip sliding-window kernels (k_iter1_s5, k_iter23_s5)
  int k1sw = 1;       // K1 variant: 1 = sliding window (k_iter1_sw), 0 = tiles (k_iter1_st)
  int g_warp = 0;     // CSR G with long rows: K3 one warp per row (k_iter3_wr)
  int small = 0;      // DIA systems of <= kSmallRows rows: one CTA per system (k_pcg_small)
  int scn = 1;        // ... of <= kClusterRows rows: one cluster of scn CTAs per system
  int smem_cn = 0;    // > 0: the shared-memory resident solver (k_pcg_smem), smem_cn CTAs of
  int smem_R = 0;     //      smem_R rows per system
  int k1pairs = 1;    // strip K1 with the coefficient stencil: two lines per step (SG_STRIP_K1_PAIRS=0: one)
  int k23 = 1;        // fused K2+K3 variant: 1 = sliding window (k_iter23_sw), 0 = tiles (k_iter23_st)
  void* sell_mem[3] = {nullptr, nullptr, nullptr};   // SELL-32 patterns of A, G, G^T
  void* sell_vals[3] = {nullptr, nullptr, nullptr};
  long long sell_total[3] = {0, 0, 0};
  int staged = 0;     // DIA with a small halo: halo-staged K1 and fused K2+K3 (k_iter1_st, k_iter23_st)
  // DIA format (0 = CSR)
  int dia_nd = 0;
  int a_sym = 0;      // DIA: A bitwise symmetric on its pattern -> lower-half reads only
  long long guard = 0;  // DIA: zero rows around every vector / diagonal
  unsigned int* d_flag = nullptr;
  void* dia_mem = nullptr;
  void* gblk_mem = nullptr;  // strip G blocks (k_strip_gblocks)
  double* dia_g = nullptr;
  double* dia_a = nullptr;
  unsigned char* dia_mask = nullptr;
  // coefficient stencil (sg_pcg_set_stencil): caller's coefficient array, the guarded copy the
  // kernels read, and whether the last solve verified A against it (cst)
  const double* coef_user = nullptr;
  double* coef = nullptr;
  int cst = 0;
  int64_t st_nx = 0, st_ny = 0;
  // fingerprints of the A, G, G^T patterns the handle was planned on (k_pattern_hash)
  unsigned long long pat_hash[3] = {0, 0, 0};
  // instrumentation: kernel launches, and (when profiling) event nodes around the kernels of
  // one non-refresh iteration per chunk -> per-kernel device time sampled inside the solve
  int64_t kernels = 0, chunks = 0;
  int64_t rebuilds = 0;  // re-plans after a pattern change (sg_pcg_rebuilds)
  int profile = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double prof_ms[3] = {0, 0, 0};
  double prof_active = 0, prof_samples = 0;
};

namespace {

template <class F>
int dispatch_pre(int pre, F f) {
  switch (pre) {
    case SG_PRECOND_IDENTITY: return f(std::integral_constant<int, SG_PRECOND_IDENTITY>());
    case SG_PRECOND_JACOBI: return f(std::integral_constant<int, SG_PRECOND_JACOBI>());
    case SG_PRECOND_LEARNED: return f(std::integral_constant<int, SG_PRECOND_LEARNED>());
  }
  set_error("unknown preconditioner kind %d", pre);
  return SG_EINVAL;
}

// f(PRE, FMT, ND, SH) over the handle's configuration.
template <class F>
int dispatch(const sg_pcg* h, F f) {
  using std::integral_constant;
  return dispatch_pre(h->pre, [&](auto P) -> int {
    if (h->dia_nd && h->a_sym) {  // DIA, A stored by its lower half (bitwise symmetric A)
      switch (h->dia_nd) {
        case 5: return f(P, integral_constant<int, 2>(), integral_constant<int, 5>(), integral_constant<bool, true>());
        case 7: return f(P, integral_constant<int, 2>(), integral_constant<int, 7>(), integral_constant<bool, true>());
        default: return f(P, integral_constant<int, 2>(), integral_constant<int, 8>(), integral_constant<bool, true>());
      }
    }
    switch (h->dia_nd) {
      case 5: return f(P, integral_constant<int, 1>(), integral_constant<int, 5>(), integral_constant<bool, true>());
      case 7: return f(P, integral_constant<int, 1>(), integral_constant<int, 7>(), integral_constant<bool, true>());
      case 1: case 2: case 3: case 4: case 6: case 8:
        return f(P, integral_constant<int, 1>(), integral_constant<int, 8>(), integral_constant<bool, true>());
      default: break;
    }
    if (h->short_rows)
      return f(P, integral_constant<int, 0>(), integral_constant<int, 0>(), integral_constant<bool, true>());
    return f(P, integral_constant<int, 0>(), integral_constant<int, 0>(), integral_constant<bool, false>());
  });
}

// Launches one iteration; returns the number of kernels launched through *nk.  With `ev`
// (profiling), external event-record nodes bracket K1, K2 and K3.
int launch_iteration(sg_pcg* h, cudaStream_t s, int par, bool refresh, cudaEvent_t* ev, int* nk) {
  return dispatch(h, [&](auto P, auto Fc, auto Nc, auto SHc) -> int {
    constexpr int PRE = decltype(P)::value;
    constexpr int FMT = decltype(Fc)::value;
    constexpr int ND = decltype(Nc)::value;
    constexpr bool SH = decltype(SHc)::value;
    const unsigned g = (unsigned)h->nblk;
    int k = 0;
    if (ev) {
      k_snapshot<<<1, 1, 0, s>>>(h->ctl); ++k;
      SG_CUDA(cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal));
    }
    constexpr int FS = FMT >= 1 ? FMT : 1;
    constexpr int NS = ND > 0 ? ND : 1;
    const bool st = FMT >= 1 && h->staged;
    const size_t tile = (size_t)PR * kRpt, H = (size_t)h->D.dia.halo;
    const unsigned gr = (unsigned)h->nrng;
    const bool strip = FMT >= 1 && ND == 5 && h->strip;
    // the streamed kernels exist with and without the row-partition logic (PART)
    auto k1_streamed = [&](auto Pc) {
      constexpr bool PT = decltype(Pc)::value;
      if (strip && FMT == 2 && h->cst && !PT && h->k1pairs)  // coefficient stencil, two lines per step
        k_iter1_s5p<<<gr, kStripC, Strip1P::SMEM, s>>>(h->D, par);
      else if (strip && FMT == 2 && h->cst && !PT)  // A from the coefficient stencil (verified per solve)
        k_iter1_s5<2, false, true><<<gr, kStripC, Strip1<2, true>::SMEM, s>>>(h->D, par);
      else if (strip) k_iter1_s5<FS, PT><<<gr, kStripC, Strip1<FS>::SMEM, s>>>(h->D, par);
      else if (st && h->k1sw && FMT == 2 && ND == 5 && h->cst && !PT) {  // A from the coefficient stencil
        if (H <= PR) k_iter1_sw<2, 5, 1, true><<<gr, PR, Sw1<2, 5, 1, true>::SMEM, s>>>(h->D, par);
        else k_iter1_sw<2, 5, 2, true><<<gr, PR, Sw1<2, 5, 2, true>::SMEM, s>>>(h->D, par);
      } else if (st && h->k1sw) {
        if (H <= PR) k_iter1_sw<FS, NS, 1, false, PT><<<gr, PR, Sw1<FS, NS, 1>::SMEM, s>>>(h->D, par);
        else k_iter1_sw<FS, NS, 2, false, PT><<<gr, PR, Sw1<FS, NS, 2>::SMEM, s>>>(h->D, par);
      } else if (H <= PR) k_iter1_st<FS, NS, 1, PT><<<g, PR, (tile + 2 * H) * sizeof(double), s>>>(h->D, par);
      else k_iter1_st<FS, NS, 2, PT><<<g, PR, (tile + 2 * H) * sizeof(double), s>>>(h->D, par);
    };
    auto k23_streamed = [&](auto Pc) {
      constexpr bool PT = decltype(Pc)::value;
      if (strip) {
        k_iter23_s5<PT><<<gr, kStripC, Strip23::SMEM, s>>>(h->D, par);
      } else if (h->k23 == 1) {
        if (H <= PR) k_iter23_sw<NS, 1, PT><<<gr, kSwThreads, Sw23<NS, 1>::SMEM, s>>>(h->D, par);
        else k_iter23_sw<NS, 2, PT><<<gr, kSwThreads, Sw23<NS, 2>::SMEM, s>>>(h->D, par);
      } else {
        if (H <= PR) k_iter23_st<NS, 1, PT><<<g, PR, (2 * tile + 6 * H) * sizeof(double), s>>>(h->D, par);
        else k_iter23_st<NS, 2, PT><<<g, PR, (2 * tile + 6 * H) * sizeof(double), s>>>(h->D, par);
      }
    };
    if (strip || st) {
      if (h->part) k1_streamed(std::true_type{});
      else k1_streamed(std::false_type{});
    } else if (FMT == 0 && !SH) {  // CSR, long rows: d' first, then one gather per nonzero
      k_pre_d<<<g, PR, 0, s>>>(h->D, par); ++k;
      k_iter1<PRE, FMT, ND, SH, true><<<g, PR, 0, s>>>(h->D, par);
    } else k_iter1<PRE, FMT, ND, SH><<<g, PR, 0, s>>>(h->D, par);
    ++k;
    if (ev) SG_CUDA(cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal));
    if ((st || strip) && !refresh && PRE == SG_PRECOND_LEARNED) {  // K2 + K3 fused
      if (h->part) k23_streamed(std::true_type{});
      else k23_streamed(std::false_type{});
      ++k;
      if (ev) {
        SG_CUDA(cudaEventRecordWithFlags(ev[2], s, cudaEventRecordExternal));
        SG_CUDA(cudaEventRecordWithFlags(ev[3], s, cudaEventRecordExternal));
      }
      SG_LAUNCH_CHECK("pcg iteration");
      *nk += k;
      return SG_OK;
    }
    if (!refresh && FMT == 0 && !SH) {
      k_pre_r<<<g, PR, 0, s>>>(h->D, par); ++k;
      if (PRE == SG_PRECOND_LEARNED && h->D.sell_on && h->g_warp) k_iter2_sell<<<g, PR, 0, s>>>(h->D, par);
      else k_iter2<PRE, FMT, ND, SH, true><<<g, PR, 0, s>>>(h->D, par);
      ++k;
    } else if (!refresh) {
      k_iter2<PRE, FMT, ND, SH><<<g, PR, 0, s>>>(h->D, par); ++k;
    } else {
      k_refresh_x<<<g, PR, 0, s>>>(h->D, par); ++k;
      k_refresh_r<FMT, ND, SH><<<g, PR, 0, s>>>(h->D, par); ++k;
      if (PRE == SG_PRECOND_LEARNED) { k_refresh_t<FMT, ND, SH><<<g, PR, 0, s>>>(h->D, par); ++k; }
    }
    if (ev) SG_CUDA(cudaEventRecordWithFlags(ev[2], s, cudaEventRecordExternal));
    if (FMT == 0 && PRE == SG_PRECOND_LEARNED && h->g_warp) k_iter3_wr<<<g, PR, 0, s>>>(h->D, par, refresh ? 1 : 0);
    else k_iter3<PRE, FMT, ND, SH><<<g, PR, 0, s>>>(h->D, par, refresh ? 1 : 0);
    ++k;
    if (ev) SG_CUDA(cudaEventRecordWithFlags(ev[3], s, cudaEventRecordExternal));
    SG_LAUNCH_CHECK("pcg iteration");
    *nk += k;
    return SG_OK;
  });
}

int get_graph(sg_pcg* h, const std::vector<int>& pattern, cudaGraphExec_t* out, int* prof_pos) {
  // profiled iteration: the first non-refresh one of the chunk
  *prof_pos = -1;
  if (h->profile)
    for (int c = 0; c < h->chunk; ++c)
      if (!pattern[c]) { *prof_pos = c; break; }
  auto it = h->graphs.find(pattern);
  if (it != h->graphs.end()) { *out = it->second; return SG_OK; }
  cudaGraph_t graph;
  SG_CUDA(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
  int rc = SG_OK, nk = 0;
  for (int c = 0; c < h->chunk && rc == SG_OK; ++c)
    rc = launch_iteration(h, h->cap_stream, c & 1, pattern[c] != 0, c == *prof_pos ? h->ev : nullptr, &nk);
  cudaError_t e = cudaStreamEndCapture(h->cap_stream, &graph);
  if (rc != SG_OK) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
  cudaGraphExec_t exec;
  SG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  cudaGraphDestroy(graph);
  h->graphs[pattern] = exec;
  h->graph_kernels[pattern] = nk;
  *out = exec;
  return SG_OK;
}

int ensure_hist(sg_pcg* h, long long need, cudaStream_t s) {
  if (need <= h->hcap) return SG_OK;
  long long cap = h->hcap ? h->hcap : 1024;
  while (cap < need) cap *= 2;
  double* nh = nullptr;
  SG_CUDA(cudaStreamSynchronize(s));
  SG_CUDA(cudaMalloc(&nh, (size_t)cap * h->S * sizeof(double)));
  if (h->hist && h->hcap)
    SG_CUDA(cudaMemcpy2DAsync(nh, cap * sizeof(double), h->hist, h->hcap * sizeof(double),
                              h->hcap * sizeof(double), h->S, cudaMemcpyDeviceToDevice, s));
  SG_CUDA(cudaStreamSynchronize(s));
  if (h->hist) SG_CUDA(cudaFree(h->hist));
  h->hist = nh;
  h->hcap = cap;
  // kernels read hist / hcap through the Ctl block, so captured graphs stay valid
  Ctl tmp;
  SG_CUDA(cudaMemcpyAsync(&tmp, h->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  tmp.hist = nh;
  tmp.hcap = cap;
  SG_CUDA(cudaMemcpyAsync(h->ctl, &tmp, sizeof(Ctl), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaStreamSynchronize(s));
  return SG_OK;
}

// Decide the DIA format: A's pattern must have <= MAXD distinct diagonals forming a symmetric
// set, G must share A's pattern (same arrays, or equal), and G^T's pattern must equal it.
int same_pattern(const int32_t* ao, const int32_t* ac, const int32_t* bo, const int32_t* bc, int64_t n,
                 bool* same, cudaStream_t s) {
  *same = true;
  if (ao == bo && ac == bc) return SG_OK;
  int32_t nnz[2] = {0, 0};
  SG_CUDA(cudaMemcpyAsync(&nnz[0], ao + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaMemcpyAsync(&nnz[1], bo + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  if (nnz[0] != nnz[1]) { *same = false; return SG_OK; }
  unsigned int* flag = nullptr;
  SG_CUDA(cudaMalloc(&flag, sizeof(unsigned int)));
  SG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned int), s));
  const int gb = 148 * 8;
  k_differ<<<gb, 256, 0, s>>>(ao, bo, n + 1, flag);
  k_differ<<<gb, 256, 0, s>>>(ac, bc, nnz[0], flag);
  SG_LAUNCH_CHECK("k_differ");
  unsigned int hf = 0;
  SG_CUDA(cudaMemcpyAsync(&hf, flag, sizeof(hf), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  cudaFree(flag);
  *same = hf == 0;
  return SG_OK;
}

int setup_dia(sg_pcg* h, const int32_t* a_offs, const int32_t* a_cols, const int32_t* g_offs,
              const int32_t* g_cols, const int32_t* gt_offs, const int32_t* gt_cols, cudaStream_t s) {
  h->dia_nd = 0;
  const int64_t n = h->n;
  if (h->pre == SG_PRECOND_LEARNED) {  // G (and G^T) must sit on A's pattern
    bool s1 = false, s2 = false;
    int rc = same_pattern(a_offs, a_cols, g_offs, g_cols, n, &s1, s);
    if (rc) return rc;
    rc = same_pattern(a_offs, a_cols, gt_offs, gt_cols, n, &s2, s);
    if (rc) return rc;
    if (!s1 || !s2) return SG_OK;
  }
  int* scratch = nullptr;
  SG_CUDA(cudaMalloc(&scratch, 32 * sizeof(int)));
  std::vector<int> init(18, INT_MIN);
  init[16] = 0;
  init[17] = 0;
  SG_CUDA(cudaMemcpyAsync(scratch, init.data(), 18 * sizeof(int), cudaMemcpyHostToDevice, s));
  const int gb = (int)(n / 256 + 1 < 148 * 8 ? n / 256 + 1 : 148 * 8);
  k_dia_offsets<<<gb, 256, 0, s>>>(a_offs, a_cols, n, scratch, scratch + 16, scratch + 17);
  SG_LAUNCH_CHECK("k_dia_offsets");
  std::vector<int> out(18);
  SG_CUDA(cudaMemcpyAsync(out.data(), scratch, 18 * sizeof(int), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  cudaFree(scratch);
  const int cnt = out[16];
  if (out[17] || cnt < 1 || cnt > MAXD) return SG_OK;
  std::vector<int> offs(out.begin(), out.begin() + cnt);
  std::sort(offs.begin(), offs.end());
  Dia dia{};
  dia.nd = cnt;
  dia.n = n;
  for (int d = 0; d < cnt; ++d) {
    dia.off[d] = offs[d];
    auto it = std::find(offs.begin(), offs.end(), -offs[d]);
    if (it == offs.end()) return SG_OK;  // offset set not symmetric
    dia.mir[d] = (int)(it - offs.begin());
  }
  // guard bands: zero rows before and after every diagonal, every vector and the mask, so
  // neighbour reads never need clamping: max |offset| rows, or the sliding-window kernel's
  // reach ((2 * ceil(H / kSwC) + 1) chunks + 16-row alignment) when halo staging is on
  long long halo = 0;
  for (int d = 0; d < cnt; ++d) halo = std::max<long long>(halo, std::abs((long long)offs[d]));
  dia.halo = (int)halo;
  const char* ns = getenv("SG_PCG_NOSTAGE");
  h->staged = (halo <= kMaxStageHalo && !(ns && ns[0] == '1')) ? 1 : 0;
  // wide 5-point grid (offsets {-W, -1, 0, 1, W}): line-strip streaming instead of 1-D rings
  dia.W = 0;
  h->strip = 0;
  if (!h->staged && cnt == 5 && !(ns && ns[0] == '1') && offs[0] == -offs[4] && offs[1] == -1 && offs[2] == 0 &&
      offs[3] == 1 && offs[4] % 16 == 0) {
    const long long W = offs[4];
    bool ok = true;
    for (int k = 0; k < h->S; ++k) ok = ok && (h->sys_start[k + 1] - h->sys_start[k]) % W == 0;
    if (ok) { dia.W = (int)W; h->strip = 1; }
  }
  long long guard = halo;
  if (h->staged) guard = std::max<long long>(guard, (2 * ((halo + kSwC - 1) / kSwC) + 1) * kSwC + 16);
  if (h->strip) guard = std::max<long long>(guard, 2LL * dia.W + 64);
  guard = (guard + 31) / 32 * 32;                // 256-byte alignment of every row-0 pointer
  const long long ld = (n + 2 * guard + 31) / 32 * 32;
  const size_t vbytes = (size_t)cnt * ld * sizeof(double);
  const size_t mbytes = (size_t)(n + 2 * guard + 64);
  SG_CUDA(cudaMalloc(&h->dia_mem, 2 * vbytes + mbytes));
  SG_CUDA(cudaMemsetAsync(h->dia_mem, 0, 2 * vbytes + mbytes, s));
  h->dia_a = reinterpret_cast<double*>(h->dia_mem) + guard;
  h->dia_g = reinterpret_cast<double*>(reinterpret_cast<char*>(h->dia_mem) + vbytes) + guard;
  h->dia_mask = reinterpret_cast<unsigned char*>(h->dia_mem) + 2 * vbytes + guard;
  dia.ld = ld;
  dia.a = h->dia_a;
  dia.g = h->dia_g;
  for (int d = 0; d < MAXD; ++d) {  // unused slots alias diagonal 0 (loaded, never masked in)
    dia.av[d] = h->dia_a + (d < cnt ? d : 0) * ld;
    dia.gv[d] = h->dia_g + (d < cnt ? d : 0) * ld;
  }
  dia.mask = h->dia_mask;
  h->D.dia = dia;
  h->dia_nd = cnt;
  h->guard = guard;
  return SG_OK;
}

// Opt the sliding-window kernels into their shared memory; blocks per SM of the (nd, nh) one.
template <int ND, int NH>
int sw_attr(int* per_sm) {
  SG_CUDA(cudaFuncSetAttribute(k_iter23_sw<ND, NH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Sw23<ND, NH>::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_sw<1, ND, NH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Sw1<1, ND, NH>::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_sw<2, ND, NH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Sw1<2, ND, NH>::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter23_sw<ND, NH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Sw23<ND, NH>::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_sw<1, ND, NH, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Sw1<1, ND, NH>::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_sw<2, ND, NH, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Sw1<2, ND, NH>::SMEM));
  if constexpr (ND == 5)
    SG_CUDA(cudaFuncSetAttribute(k_iter1_sw<2, 5, NH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)Sw1<2, 5, NH, true>::SMEM));
  SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_iter23_sw<ND, NH>, kSwThreads, Sw23<ND, NH>::SMEM));
  if (*per_sm < 1) *per_sm = 1;
  return SG_OK;
}

// One cluster of CN 1024-thread CTAs per system (k_pcg_small<..., CN>): can the GPU co-schedule it?
template <int CN>
int cluster_fits_t(int* nclusters) {
  auto kern = k_pcg_small<SG_PRECOND_LEARNED, 2, 5, CN>;
  if (CN > 8) SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(CN);
  c.blockDim = dim3(kSmallThreads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CN;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  c.attrs = at;
  c.numAttrs = 1;
  SG_CUDA(cudaOccupancyMaxActiveClusters(nclusters, kern, &c));
  return SG_OK;
}
int cluster_fits(int cn, int* nclusters) {
  switch (cn) {
    case 2: return cluster_fits_t<2>(nclusters);
    case 4: return cluster_fits_t<4>(nclusters);
    case 8: return cluster_fits_t<8>(nclusters);
    default: return cluster_fits_t<16>(nclusters);
  }
}

template <int PRE, int FMT, int ND, int CN>
int launch_cluster(sg_pcg* h, int chunk, long long period, cudaStream_t s) {
  auto kern = k_pcg_small<PRE, FMT, ND, CN>;
  if (CN > 8) SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3((unsigned)(h->S * CN));
  c.blockDim = dim3(kSmallThreads);
  c.dynamicSmemBytes = 0;
  c.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CN;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  c.attrs = at;
  c.numAttrs = 1;
  SG_CUDA(cudaLaunchKernelEx(&c, kern, h->D, chunk, period));
  return SG_OK;
}

constexpr size_t kSmemSysMax = 227 * 1024 - 4096;  // dynamic shared memory of one k_pcg_smem CTA (+ its static)

template <int CN>
int smem_fits_t(size_t bytes, int* nclusters) {
  auto kern = k_pcg_smem<SG_PRECOND_LEARNED, 1, 8, CN>;
  SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemSysMax));
  if (CN > 8) SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  if (CN == 1) {
    int nb = 0;
    SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kSmallThreads, bytes));
    *nclusters = nb;
    return SG_OK;
  }
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(CN);
  c.blockDim = dim3(kSmallThreads);
  c.dynamicSmemBytes = bytes;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CN;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  c.attrs = at;
  c.numAttrs = 1;
  SG_CUDA(cudaOccupancyMaxActiveClusters(nclusters, kern, &c));
  return SG_OK;
}
int smem_fits(int cn, size_t bytes, int* nclusters) {
  switch (cn) {
    case 1: return smem_fits_t<1>(bytes, nclusters);
    case 2: return smem_fits_t<2>(bytes, nclusters);
    case 4: return smem_fits_t<4>(bytes, nclusters);
    case 8: return smem_fits_t<8>(bytes, nclusters);
    default: return smem_fits_t<16>(bytes, nclusters);
  }
}

template <int PRE, int FMT, int ND, int CN>
int launch_smem(sg_pcg* h, int chunk, long long period, cudaStream_t s) {
  auto kern = k_pcg_smem<PRE, FMT, ND, CN>;
  constexpr int NA = FMT == 2 ? ND / 2 + 1 : ND;
  const size_t bytes = smem_sys_bytes(h->smem_R, h->D.dia.halo, NA, ND);
  SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  if (CN > 8) SG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3((unsigned)(h->S * CN));
  c.blockDim = dim3(kSmallThreads);
  c.dynamicSmemBytes = bytes;
  c.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CN;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  c.attrs = at;
  c.numAttrs = CN > 1 ? 1 : 0;
  SG_CUDA(cudaLaunchKernelEx(&c, kern, h->D, chunk, period, h->smem_R));
  return SG_OK;
}

int strip_setup(int* per_sm) {
  SG_CUDA(cudaFuncSetAttribute(k_iter23_s5<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Strip23::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter23_s5<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Strip23::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_s5<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Strip1<1>::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_s5<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Strip1<2>::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_s5<2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)Strip1<2, true>::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_s5p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Strip1P::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_s5<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Strip1<1>::SMEM));
  SG_CUDA(cudaFuncSetAttribute(k_iter1_s5<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Strip1<2>::SMEM));
  SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_iter23_s5<false>, kStripC, Strip23::SMEM));
  if (*per_sm < 1) *per_sm = 1;
  return SG_OK;
}

int sw_setup(int nd, int nh, int* per_sm) {
  const int ns = nd == 5 ? 5 : (nd == 7 ? 7 : 8);
  if (ns == 5) return nh == 1 ? sw_attr<5, 1>(per_sm) : sw_attr<5, 2>(per_sm);
  if (ns == 7) return nh == 1 ? sw_attr<7, 1>(per_sm) : sw_attr<7, 2>(per_sm);
  return nh == 1 ? sw_attr<8, 1>(per_sm) : sw_attr<8, 2>(per_sm);
}


// SELL-32 copy of a CSR pattern (slice offsets + column indices); values are filled per solve.
int sell_pattern(sg_pcg* h, const int32_t* offs, const int32_t* cols, cudaStream_t s, Sell* out, void** mem_out,
                 long long* total_out) {
  const int64_t n = h->n;
  std::vector<int32_t> ho(n + 1);
  SG_CUDA(cudaMemcpyAsync(ho.data(), offs, (n + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  const int64_t ns = (n + 31) / 32;
  std::vector<long long> sb(ns + 1, 0);
  for (int64_t sl = 0; sl < ns; ++sl) {
    int mx = 0;
    for (int64_t r = sl * 32; r < std::min<int64_t>(n, sl * 32 + 32); ++r) mx = std::max(mx, ho[r + 1] - ho[r]);
    sb[sl + 1] = sb[sl] + 32LL * mx;
  }
  const long long total = sb[ns];
  char* mem = nullptr;
  const size_t bytes = (ns + 1) * sizeof(long long) + (size_t)total * sizeof(int32_t) + 512;
  SG_CUDA(cudaMalloc(&mem, bytes));
  long long* d_sb = reinterpret_cast<long long*>(mem);
  int32_t* d_cols = reinterpret_cast<int32_t*>(mem + (((ns + 1) * sizeof(long long) + 255) / 256) * 256);
  SG_CUDA(cudaMemcpyAsync(d_sb, sb.data(), (ns + 1) * sizeof(long long), cudaMemcpyHostToDevice, s));
  const int gb = (int)std::min<int64_t>(n / 256 + 1, 148 * 16);
  k_csr_to_sell<<<gb, 256, 0, s>>>(n, offs, cols, nullptr, d_sb, d_cols, nullptr);
  SG_LAUNCH_CHECK("k_csr_to_sell (pattern)");
  out->sbase = d_sb;
  out->cols = d_cols;
  out->offs = offs;
  *mem_out = mem;
  *total_out = total;
  return SG_OK;
}

int setup_sell(sg_pcg* h, const int32_t* a_offs, const int32_t* a_cols, const int32_t* g_offs,
               const int32_t* g_cols, const int32_t* gt_offs, const int32_t* gt_cols, cudaStream_t s) {
  int rc = sell_pattern(h, a_offs, a_cols, s, &h->D.sa, &h->sell_mem[0], &h->sell_total[0]);
  if (rc) return rc;
  (void)g_offs; (void)g_cols;
  if (h->pre == SG_PRECOND_LEARNED &&
      (rc = sell_pattern(h, gt_offs, gt_cols, s, &h->D.sgt, &h->sell_mem[2], &h->sell_total[2])))
    return rc;
  for (int k = 0; k < 3; ++k)
    if (h->sell_total[k] > 0) SG_CUDA(cudaMalloc(&h->sell_vals[k], (size_t)h->sell_total[k] * sizeof(double) + 64));
  h->D.sa.vals = static_cast<double*>(h->sell_vals[0]);
  h->D.sg.vals = static_cast<double*>(h->sell_vals[1]);
  h->D.sgt.vals = static_cast<double*>(h->sell_vals[2]);
  // G's rows are summed in numpy's pairwise order, whose 8-wide leaf blocks read better from the
  // row-contiguous CSR (measured at C4: 3.8 ms CSR vs 5.0 ms SELL); A and G^T use SELL
  h->D.sell_on = 1;
  return SG_OK;
}
}  // namespace

namespace {
// d_flag block: [0] A not bitwise symmetric, [1] stencil mismatch, [2] unmatched DIA entry,
// [3] unused; bytes 16..39: the three pattern fingerprints of this solve.
constexpr int kFlagBytes = 40;

int pattern_hashes(sg_pcg* h, cudaStream_t s) {
  SG_CUDA(cudaMemsetAsync(h->d_flag, 0, kFlagBytes, s));
  unsigned long long* out = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(h->d_flag) + 16);
  const int gb = (int)(h->n / 1024 + 1 < 148 * 8 ? h->n / 1024 + 1 : 148 * 8);
  k_pattern_hash<<<gb, 256, 0, s>>>(h->D.a_offs, h->D.a_cols, h->n, 0x51ull, out);
  if (h->pre == SG_PRECOND_LEARNED) {
    k_pattern_hash<<<gb, 256, 0, s>>>(h->D.g_offs, h->D.g_cols, h->n, 0x52ull, out + 1);
    k_pattern_hash<<<gb, 256, 0, s>>>(h->D.gt_offs, h->D.gt_cols, h->n, 0x53ull, out + 2);
  }
  SG_LAUNCH_CHECK("k_pattern_hash");
  h->kernels += h->pre == SG_PRECOND_LEARNED ? 3 : 1;
  return SG_OK;
}

// Re-plan a handle whose patterns changed under it: a fresh handle on the same pointers takes
// over (user settings carried), the old resources are released.
int rebuild(sg_pcg* h, cudaStream_t s) {
  if (h->part) {
    set_error("the sparsity pattern of a row-partitioned PCG handle changed; create a new handle");
    return SG_EINVAL;
  }
  sg_pcg* nh = nullptr;
  int rc = sg_pcg_create(&nh, h->S, h->sys_start.data(), h->D.a_offs, h->D.a_cols, h->D.a_vals, h->pre,
                         h->D.g_offs, h->D.g_cols, h->D.g_vals, h->D.gt_offs, h->D.gt_cols, h->D.gt_vals,
                         h->D.inv_diag, h->eps, s);
  if (rc) return rc;
  nh->profile = h->profile;
  nh->kernels = h->kernels;
  nh->chunks = h->chunks;
  for (int k = 0; k < 3; ++k) nh->prof_ms[k] = h->prof_ms[k];
  nh->prof_active = h->prof_active;
  nh->prof_samples = h->prof_samples;
  nh->rebuilds = h->rebuilds + 1;
  const double* cu = h->coef_user;
  const int64_t nx = h->st_nx, ny = h->st_ny;
  std::swap(*h, *nh);
  sg_pcg_destroy(nh);
  if (cu) {
    int32_t ok = 0;
    rc = sg_pcg_set_stencil(h, cu, nx, ny, &ok);
  }
  return rc;
}
}  // namespace

extern "C" int sg_pcg_create(sg_pcg** out, int32_t n_systems, const int64_t* sys_row_start_host,
                             const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                             int precond_kind, const int32_t* g_offs, const int32_t* g_cols,
                             const double* g_vals, const int32_t* gt_offs, const int32_t* gt_cols,
                             const double* gt_vals, const double* inv_diag, double epsilon,
                             void* stream) {
  if (n_systems < 1) { set_error("need at least one system"); return SG_EINVAL; }
  if (precond_kind < 0 || precond_kind > 2) { set_error("unknown preconditioner kind"); return SG_EINVAL; }
  if (precond_kind == SG_PRECOND_LEARNED && epsilon < 0.0) { set_error("epsilon must be nonnegative"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  sg_pcg* h = new sg_pcg();
  {
    int dev = 0;
    SG_CUDA(cudaGetDevice(&dev));
    SG_CUDA(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  h->S = n_systems;
  h->pre = precond_kind;
  h->eps = epsilon;
  h->sys_start.assign(sys_row_start_host, sys_row_start_host + n_systems + 1);
  h->n = h->sys_start.back();
  for (int k = 0; k < n_systems; ++k)
    if (h->sys_start[k + 1] <= h->sys_start[k]) {
      delete h;
      set_error("every system needs at least one row");
      return SG_EINVAL;
    }
  // storage format first: it fixes the tile size
  {  // longest row of every matrix the loop touches -> SHORT CSR kernels when all are <= 8
    unsigned int* mx = nullptr;
    SG_CUDA(cudaMalloc(&mx, sizeof(unsigned int)));
    SG_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned int), s));
    const int64_t n = h->n;
    const int gb = (int)(n / 256 + 1 < 148 * 8 ? n / 256 + 1 : 148 * 8);
    k_max_row<<<gb, 256, 0, s>>>(a_offs, n, mx);
    if (precond_kind == SG_PRECOND_LEARNED) {
      k_max_row<<<gb, 256, 0, s>>>(g_offs, n, mx);
      k_max_row<<<gb, 256, 0, s>>>(gt_offs, n, mx);
    }
    SG_LAUNCH_CHECK("k_max_row");
    unsigned int hm = 0;
    SG_CUDA(cudaMemcpyAsync(&hm, mx, sizeof(hm), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    cudaFree(mx);
    h->short_rows = hm <= 8 ? 1 : 0;
  }
  {
    int rc = setup_dia(h, a_offs, a_cols, g_offs, g_cols, gt_offs, gt_cols, s);
    if (rc) { delete h; return rc; }
  }
  const int tile = h->dia_nd ? PR * kRpt : PR;
  std::vector<long long> blk_r0;
  std::vector<int> blk_sys, sys_blk0;
  std::vector<long long> sys_r1;
  for (int k = 0; k < n_systems; ++k) {
    sys_blk0.push_back((int)blk_r0.size());
    const int64_t a = h->sys_start[k], b = h->sys_start[k + 1];
    for (int64_t r = a; r < b; r += tile) { blk_r0.push_back(r); blk_sys.push_back(k); }
    sys_r1.push_back(b);
  }
  sys_blk0.push_back((int)blk_r0.size());
  h->nblk = (int)blk_r0.size();
  // sliding-window ranges (halo-staged DIA): m ranges per system, m chosen against the number of
  // co-resident CTAs (whole waves) and the 4*NH-chunk warm-up every range pays
  long long rng_len = 1;
  if (h->staged) {
    const int nh = h->D.dia.halo <= kSwC ? 1 : 2;
    int per_sm = 1;
    int rc = sw_setup(h->dia_nd, nh, &per_sm);
    if (rc) { delete h; return rc; }
    const long long resident = (long long)h->num_sms * per_sm;
    long long maxrows = 1;
    for (int k = 0; k < n_systems; ++k) maxrows = std::max<long long>(maxrows, h->sys_start[k + 1] - h->sys_start[k]);
    double best = 1e300;
    const long long mmax = std::max<long long>(1, std::min<long long>(256, maxrows / kSwC));  // ranges >= C rows
    for (long long m = 1; m <= mmax; ++m) {
      const long long len = (maxrows + m - 1) / m;
      const double waves = (double)((n_systems * m + resident - 1) / resident);
      const double cost = waves * (double)(len + 4LL * nh * kSwC);
      if (cost < best * 0.999) { best = cost; rng_len = len; }
    }
    const char* rl = getenv("SG_SW_RANGE");
    if (rl && atoll(rl) > 0) rng_len = atoll(rl);
  } else if (h->strip) {  // (strip, line range) units; rng_len counts LINES
    int per_sm = 1;
    int rc = strip_setup(&per_sm);
    if (rc) { delete h; return rc; }
    const long long resident = (long long)h->num_sms * per_sm;
    const long long W = h->D.dia.W, nstrip = (W + kStripC - 1) / kStripC;
    long long maxl = 1;
    for (int k = 0; k < n_systems; ++k) maxl = std::max<long long>(maxl, (h->sys_start[k + 1] - h->sys_start[k]) / W);
    double best = 1e300;
    for (long long m = 1; m <= std::min<long long>(maxl, 1024); ++m) {
      const long long len = (maxl + m - 1) / m;
      const double waves = (double)((n_systems * nstrip * m + resident - 1) / resident);
      const double cost = waves * (double)(len + 4);
      if (cost < best * 0.999) { best = cost; rng_len = len; }
    }
    const char* rl = getenv("SG_SW_RANGE");
    if (rl && atoll(rl) > 0) rng_len = atoll(rl);
    if (h->pre == SG_PRECOND_LEARNED) {  // G strip blocks: every system's lines + 4 zero lines, per strip
      const long long L = h->n / W + 4LL * n_systems;
      SG_CUDA(cudaMalloc(&h->gblk_mem, (size_t)(nstrip * L) * kStripBB));
      h->D.gblk = static_cast<const unsigned char*>(h->gblk_mem);
      h->D.gblk_L = L;
    }
  } else {
    rng_len = 1LL << 62;
  }
  std::vector<long long> rng_r0;
  std::vector<int> rng_sys, sys_rng0;
  for (int k = 0; k < n_systems; ++k) {
    sys_rng0.push_back((int)rng_r0.size());
    if (h->strip) {
      const long long W = h->D.dia.W, nl = (h->sys_start[k + 1] - h->sys_start[k]) / W;
      for (long long y = 0; y < nl; y += rng_len)
        for (long long x = 0; x < W; x += kStripC) {
          rng_r0.push_back(h->sys_start[k] + y * W + x);
          rng_sys.push_back(k);
        }
      continue;
    }
    for (int64_t r = h->sys_start[k]; r < h->sys_start[k + 1]; r += rng_len) {
      rng_r0.push_back(r);
      rng_sys.push_back(k);
    }
  }
  sys_rng0.push_back((int)rng_r0.size());
  h->nrng = (int)rng_r0.size();
  const int64_t n = h->n, S = n_systems, nb = h->nblk > 0 ? h->nblk : 1;
  Carve c(nullptr);
  c.take<long long>(nb); c.take<int>(nb); c.take<int>(S + 1); c.take<long long>(S);
  c.take<long long>(h->nrng); c.take<int>(h->nrng); c.take<int>(S + 1);
  c.take<long long>(S); c.take<long long>(S);
  const int64_t gv = h->guard;  // zero guard rows around every vector (DIA neighbour reads)
  for (int v = 0; v < 9; ++v) c.take<double>(n + 2 * gv + 2);
  const int64_t npart = std::max<int64_t>(nb, h->nrng);  // per-CTA partials: tiles or ranges
  c.take<double>(2 * npart); c.take<unsigned int>(S); c.take<SysState>(S); c.take<Ctl>(1);
  int e = cudaMalloc(&h->mem, c.off);
  if (e != cudaSuccess) { delete h; return cuda_fail((cudaError_t)e, "cudaMalloc(pcg workspace)"); }
  Carve m(h->mem);
  long long* d_blk_r0 = m.take<long long>(nb);
  int* d_blk_sys = m.take<int>(nb);
  int* d_sys_blk0 = m.take<int>(S + 1);
  long long* d_sys_r1 = m.take<long long>(S);
  long long* d_rng_r0 = m.take<long long>(h->nrng);
  int* d_rng_sys = m.take<int>(h->nrng);
  int* d_sys_rng0 = m.take<int>(S + 1);
  long long* d_own0 = m.take<long long>(S);
  long long* d_own1 = m.take<long long>(S);
  double* vec[9];
  for (int v = 0; v < 9; ++v) vec[v] = m.take<double>(n + 2 * gv + 2) + gv;
  double* part = m.take<double>(2 * npart);
  unsigned int* counter = m.take<unsigned int>(S);
  h->st = m.take<SysState>(S);
  h->ctl = m.take<Ctl>(1);
  SG_CUDA(cudaMemsetAsync(h->mem, 0, c.off, s));  // guards (and everything else) start at zero
  if (h->nblk) {
    SG_CUDA(cudaMemcpyAsync(d_blk_r0, blk_r0.data(), blk_r0.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(d_blk_sys, blk_sys.data(), blk_sys.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  }
  SG_CUDA(cudaMemcpyAsync(d_sys_blk0, sys_blk0.data(), sys_blk0.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(d_sys_r1, sys_r1.data(), sys_r1.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(d_rng_r0, rng_r0.data(), rng_r0.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(d_rng_sys, rng_sys.data(), rng_sys.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(d_sys_rng0, sys_rng0.data(), sys_rng0.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  // owned rows = the whole system until sg_pcg_set_partition / sg_pcg_set_peers say otherwise
  SG_CUDA(cudaMemcpyAsync(d_own0, h->sys_start.data(), S * sizeof(long long), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(d_own1, h->sys_start.data() + 1, S * sizeof(long long), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemsetAsync(counter, 0, S * sizeof(unsigned int), s));
  Dev& D = h->D;
  D.blk_r0 = d_blk_r0; D.blk_sys = d_blk_sys; D.sys_blk0 = d_sys_blk0; D.sys_r1 = d_sys_r1;
  D.tile = tile;
  D.rng_r0 = d_rng_r0; D.rng_sys = d_rng_sys; D.sys_rng0 = d_sys_rng0; D.rng_len = rng_len;
  D.own0 = d_own0; D.own1 = d_own1; D.part = 0; D.nsys = (int)S;
  D.a_offs = a_offs; D.a_cols = a_cols; D.a_vals = a_vals;
  D.g_offs = g_offs; D.g_cols = g_cols; D.g_vals = g_vals;
  D.gt_offs = gt_offs; D.gt_cols = gt_cols; D.gt_vals = gt_vals;
  D.inv_diag = inv_diag;
  D.b = vec[0]; D.x = vec[1]; D.r0 = vec[2]; D.r1 = vec[3]; D.d0 = vec[4]; D.d1 = vec[5];
  D.q = vec[6]; D.s = vec[7]; D.t = vec[8];
  D.pp = part; D.counter = counter; D.st = h->st; D.ctl = h->ctl;
  D.sell_on = 0;
  D.xdefer = 0;
  if (!h->dia_nd && !h->short_rows) {  // long CSR rows: SELL-32 copies (coalesced row walks)
    int32_t nz = 0;
    SG_CUDA(cudaMemcpyAsync(&nz, a_offs + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    const char* sv = getenv("SG_PCG_SELL");
    if (!(sv && sv[0] == '0') && n > 0 && (double)nz / (double)n >= 12.0) {
      int rc = setup_sell(h, a_offs, a_cols, g_offs, g_cols, gt_offs, gt_cols, s);
      if (rc) { sg_pcg_destroy(h); return rc; }
    }
    if (precond_kind == SG_PRECOND_LEARNED && n > 0) {  // G rows of >= 32 entries: a warp per row
      int32_t gz = 0;
      SG_CUDA(cudaMemcpyAsync(&gz, g_offs + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      SG_CUDA(cudaStreamSynchronize(s));
      const char* wv = getenv("SG_PCG_GWARP");
      h->g_warp = !(wv && wv[0] == '0') && (double)gz / (double)n >= 32.0;
    }
  }
  {
    const char* pv = getenv("SG_STRIP_K1_PAIRS");
    h->k1pairs = (pv && pv[0] == '0') ? 0 : 1;
  }
  SG_CUDA(cudaHostAlloc(&h->pinned_active, 2 * sizeof(unsigned int), cudaHostAllocDefault));
  SG_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  for (int k = 0; k < 4; ++k) SG_CUDA(cudaEventCreate(&h->ev[k]));
  if (h->staged) {
    const char* kv = getenv("SG_PCG_K23");
    // the sliding window takes the mirror of diagonal d as ND-1-d: only for full diagonal sets
    // ring_nb / the compile-time mirror ND-1-d need a sorted set with off[d] == -off[ND-1-d]
    // (and 0 in the middle for odd ND); setup_dia guarantees it, checked here where it is relied on
    bool mirrored = true;
    for (int d = 0; d < h->dia_nd; ++d) mirrored = mirrored && h->D.dia.off[d] == -h->D.dia.off[h->dia_nd - 1 - d];
    const bool full = mirrored && (h->dia_nd == 5 || h->dia_nd == 7 || h->dia_nd == 8);
    h->k23 = (kv && kv[0] == 't') || !full ? 0 : 1;
    const char* k1v = getenv("SG_PCG_K1");
    h->k1sw = (k1v && k1v[0] == 't') || !mirrored || !(h->dia_nd == 5 || h->dia_nd == 7) ? 0 : 1;
    // deferred x update: both sliding-window kernels, learned factor, one rank
    const char* sv2 = getenv("SG_PCG_SMALL");
    long long maxrows = 0;
    for (int k = 0; k < n_systems; ++k) maxrows = std::max<long long>(maxrows, h->sys_start[k + 1] - h->sys_start[k]);
    const bool sm_on = !(sv2 && sv2[0] == '0');
    h->small = sm_on && maxrows <= kSmallRows ? 1 : 0;
    h->scn = 1;
    h->smem_cn = 0;
    const char* mv = getenv("SG_PCG_SMEM");
    if (sm_on && !(mv && mv[0] == '0') && true) {
      // the whole system in shared memory: the fewest CTAs that hold it with one row per thread,
      // else with two
      const int H = h->D.dia.halo, nd = h->dia_nd;
      for (int pass = 0; pass < 2 && !h->smem_cn; ++pass)
      for (int cn = 1; cn <= 16; cn *= 2) {
        const int R = (int)((maxrows + cn - 1) / cn);
        if (R > (pass + 1) * kSmallThreads || (cn > 1 && R < H)) continue;
        const size_t bytes = smem_sys_bytes(R, H, nd, nd);
        if (bytes > kSmemSysMax) continue;
        int nclu = 1;
        if (smem_fits(cn, bytes, &nclu) != SG_OK || nclu < 1) { cudaGetLastError(); continue; }
        h->smem_cn = cn;
        h->smem_R = R;
        break;
      }
      if (h->smem_cn) h->small = 1;
    }
    const char* cv = getenv("SG_PCG_CLUSTER");
    if (sm_on && !h->small && !h->smem_cn && maxrows <= kClusterRows && !(cv && cv[0] == '0')) {
      // mid-size systems: one thread-block cluster per system, ~2048 rows per CTA
      int cn = 2;
      while (cn < 16 && (long long)cn * 2048 < maxrows) cn *= 2;
      for (; cn >= 2; cn /= 2) {
        int nclu = 0;
        if (cluster_fits(cn, &nclu) == SG_OK && nclu > 0) break;
      }
      if (cn >= 2) { h->small = 1; h->scn = cn; }
      cudaGetLastError();
    }
    const char* xv = getenv("SG_PCG_XDEFER");
    h->D.xdefer = (xv && xv[0] == '1') && h->k1sw && h->k23 == 1 && !h->strip &&
                  h->pre == SG_PRECOND_LEARNED ? 1 : 0;
  }
  SG_CUDA(cudaMalloc(&h->d_flag, kFlagBytes));
  {
    const int64_t k0 = h->kernels;
    int rc = pattern_hashes(h, s);
    if (rc) { sg_pcg_destroy(h); return rc; }
    h->kernels = k0;
    unsigned char fb[kFlagBytes];
    SG_CUDA(cudaMemcpyAsync(fb, h->d_flag, kFlagBytes, cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    memcpy(h->pat_hash, fb + 16, sizeof(h->pat_hash));
  }
  SG_CUDA(cudaStreamSynchronize(s));
  *out = h;
  return SG_OK;
}

extern "C" int sg_pcg_solve(sg_pcg* h, const double* b, double* x, const sg_solve_config* cfg,
                            sg_solve_result* results_host, int64_t* elapsed_ns_host, void* stream) {
  if (!h || !cfg) { set_error("null handle or config"); return SG_EINVAL; }
  if (!(cfg->rtol > 0.0)) { set_error("rtol must be positive"); return SG_EINVAL; }
  if (cfg->refresh_period < 1) { set_error("residual refresh period must be at least 1"); return SG_EINVAL; }
  cudaStream_t s = as_stream(stream);
  cudaEvent_t e0, e1;
  SG_CUDA(cudaEventCreate(&e0));
  SG_CUDA(cudaEventCreate(&e1));
  SG_CUDA(cudaEventRecord(e0, s));
  const int64_t period = cfg->refresh_period;
  int chunk = period <= 64 ? (int)(period % 2 == 0 ? period : 2 * period) : 64;
  if (chunk != h->chunk || period != h->period) {
    for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
    h->graphs.clear();
    h->graph_kernels.clear();
    h->chunk = chunk;
    h->period = period;
  }
  // the patterns the handle was planned on must still be the caller's (see k_pattern_hash)
  {
    int rc0 = pattern_hashes(h, s);
    if (rc0) return rc0;
  }
  // DIA: (re)build the diagonal-major values from the CSR arrays (values may change between
  // solves: a new G from the GNN, a refilled A)
  if (h->dia_nd) {
    const int gb = (int)(h->n / 256 + 1 < 148 * 16 ? h->n / 256 + 1 : 148 * 16);
    k_csr_to_dia<<<gb, 256, 0, s>>>(h->D.a_offs, h->D.a_cols, h->D.a_vals, h->n, h->D.dia, h->dia_a, h->dia_mask,
                                    h->d_flag + 2);
    if (h->pre == SG_PRECOND_LEARNED)
      k_csr_to_dia<<<gb, 256, 0, s>>>(h->D.g_offs, h->D.g_cols, h->D.g_vals, h->n, h->D.dia, h->dia_g, nullptr,
                                      h->d_flag + 2);
    if (h->gblk_mem) {
      k_strip_gblocks<<<dim3(148 * 4, (unsigned)h->S), 256, 0, s>>>(h->D, static_cast<unsigned char*>(h->gblk_mem));
      SG_LAUNCH_CHECK("k_strip_gblocks");
      h->kernels += 1;
    }
    k_dia_symcheck<<<gb, 256, 0, s>>>(h->D.dia, h->d_flag);
    SG_LAUNCH_CHECK("k_csr_to_dia / k_dia_symcheck");
    h->kernels += h->pre == SG_PRECOND_LEARNED ? 3 : 2;
    if (h->coef) {  // this solve's coefficients -> the guarded copy; verify A against them
      SG_CUDA(cudaMemcpyAsync(h->coef, h->coef_user, h->n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      k_stencil_check<<<gb, 256, 0, s>>>(h->D.dia, h->coef, h->D.ihx2, h->D.ihy2, h->d_flag + 1);
      SG_LAUNCH_CHECK("k_stencil_check");
      h->kernels += 1;
    }
  }
  unsigned char fb[kFlagBytes];
  SG_CUDA(cudaMemcpyAsync(fb, h->d_flag, kFlagBytes, cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  unsigned int flags[4];
  unsigned long long hs[3];
  memcpy(flags, fb, sizeof(flags));
  memcpy(hs, fb + 16, sizeof(hs));
  if (hs[0] != h->pat_hash[0] || hs[1] != h->pat_hash[1] || hs[2] != h->pat_hash[2]) {
    // the index buffers were refilled with another pattern: re-plan the handle, solve again
    int rc0 = rebuild(h, s);
    if (rc0) return rc0;
    SG_CUDA(cudaEventDestroy(e0));
    SG_CUDA(cudaEventDestroy(e1));
    return sg_pcg_solve(h, b, x, cfg, results_host, elapsed_ns_host, stream);
  }
  if (h->dia_nd && flags[2]) {
    set_error("a stored entry lies outside the handle's diagonal set (pattern changed without a rebuild)");
    return SG_EINVAL;
  }
  if (h->dia_nd) {
    const int sym = flags[0] ? 0 : 1;
    const int cst = (h->coef && sym && !flags[1]) ? 1 : 0;
    if (sym != h->a_sym || cst != h->cst) {  // kernel variant changes: captured graphs are stale
      for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
      h->graphs.clear();
      h->graph_kernels.clear();
      h->a_sym = sym;
      h->cst = cst;
    }
  }
  if (h->D.sell_on) {  // SELL-32 values of A, G, G^T (they may change between solves)
    const int gb = (int)(h->n / 256 + 1 < 148 * 16 ? h->n / 256 + 1 : 148 * 16);
    k_csr_to_sell<<<gb, 256, 0, s>>>(h->n, h->D.a_offs, nullptr, h->D.a_vals, h->D.sa.sbase, nullptr,
                                     const_cast<double*>(h->D.sa.vals));
    if (h->pre == SG_PRECOND_LEARNED)
      k_csr_to_sell<<<gb, 256, 0, s>>>(h->n, h->D.gt_offs, nullptr, h->D.gt_vals, h->D.sgt.sbase, nullptr,
                                       const_cast<double*>(h->D.sgt.vals));
    SG_LAUNCH_CHECK("k_csr_to_sell");
    h->kernels += h->pre == SG_PRECOND_LEARNED ? 2 : 1;
  }
  // per-system state
  std::vector<SysState> st(h->S);
  for (int k = 0; k < h->S; ++k) {
    memset(&st[k], 0, sizeof(SysState));
    const int64_t ns = h->sys_start[k + 1] - h->sys_start[k];
    st[k].max_iters = cfg->max_iters < 0 ? 20 * (h->part ? h->part_n : ns) : cfg->max_iters;
    st[k].status = ST_RUN;
  }
  SG_CUDA(cudaMemcpyAsync(h->st, st.data(), st.size() * sizeof(SysState), cudaMemcpyHostToDevice, s));
  int rc = ensure_hist(h, cfg->track_history ? 2 * (long long)chunk + 2 : 1, s);
  if (rc) return rc;
  Ctl ctl{};
  ctl.rtol = cfg->rtol;
  ctl.eps = h->eps;
  ctl.hist = h->hist;
  ctl.hcap = h->hcap;
  ctl.track = cfg->track_history ? 1 : 0;
  ctl.delta_mode = cfg->termination == 1 ? 1 : 0;
  ctl.n_active = (unsigned)h->S;
  SG_CUDA(cudaMemcpyAsync(h->ctl, &ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s));
  if (h->n > 0) SG_CUDA(cudaMemcpyAsync(h->D.b, b, h->n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  // setup
  const unsigned g = (unsigned)h->nblk;
  rc = dispatch(h, [&](auto P, auto Fc, auto Nc, auto SHc) -> int {
    constexpr int PRE = decltype(P)::value;
    constexpr int FMT = decltype(Fc)::value;
    constexpr int ND = decltype(Nc)::value;
    constexpr bool SH = decltype(SHc)::value;
    k_setup1<PRE, FMT, ND, SH><<<g, PR, 0, s>>>(h->D);
    k_setup2<PRE, FMT, ND, SH><<<g, PR, 0, s>>>(h->D);
    SG_LAUNCH_CHECK("pcg setup");
    return SG_OK;
  });
  if (rc) return rc;
  h->kernels += 2;
  // device-resident loop: graphs of `chunk` iterations, poll the active count between chunks
  int64_t it = 0;
  int prev_prof = -1;
  for (;;) {
    SG_CUDA(cudaMemcpyAsync(h->pinned_active, &h->ctl->n_active, 2 * sizeof(unsigned int),
                            cudaMemcpyDeviceToHost, s));
    SG_CUDA(cudaStreamSynchronize(s));
    if (prev_prof >= 0) {  // harvest the event nodes of the chunk that just finished
      float t1 = 0.f, t2 = 0.f, t3 = 0.f;
      if (cudaEventElapsedTime(&t1, h->ev[0], h->ev[1]) == cudaSuccess &&
          cudaEventElapsedTime(&t2, h->ev[1], h->ev[2]) == cudaSuccess &&
          cudaEventElapsedTime(&t3, h->ev[2], h->ev[3]) == cudaSuccess && h->pinned_active[1] > 0) {
        h->prof_ms[0] += t1; h->prof_ms[1] += t2; h->prof_ms[2] += t3;
        h->prof_active += h->pinned_active[1];
        h->prof_samples += 1;
      }
      cudaGetLastError();  // an unrecorded event must not poison later launch checks
    }
    if (h->pinned_active[0] == 0) break;
    if (cfg->track_history) {
      rc = ensure_hist(h, it + chunk + 2, s);
      if (rc) return rc;
    }
    if (h->small) {  // one CTA per system runs `chunk` whole iterations
      rc = dispatch(h, [&](auto P, auto Fc, auto Nc, auto) -> int {
        constexpr int PRE = decltype(P)::value;
        constexpr int FMT = decltype(Fc)::value;
        constexpr int ND = decltype(Nc)::value;
        if constexpr (FMT >= 1) {
          if (h->smem_cn) {
            int lrc = SG_OK;
            switch (h->smem_cn) {
              case 1: lrc = launch_smem<PRE, FMT, ND, 1>(h, chunk, period, s); break;
              case 2: lrc = launch_smem<PRE, FMT, ND, 2>(h, chunk, period, s); break;
              case 4: lrc = launch_smem<PRE, FMT, ND, 4>(h, chunk, period, s); break;
              case 8: lrc = launch_smem<PRE, FMT, ND, 8>(h, chunk, period, s); break;
              default: lrc = launch_smem<PRE, FMT, ND, 16>(h, chunk, period, s); break;
            }
            if (lrc) return lrc;
          } else if (h->scn <= 1) {
            k_pcg_small<PRE, FMT, ND><<<(unsigned)h->S, kSmallThreads, 0, s>>>(h->D, chunk, period);
          } else {
            int lrc = SG_OK;
            switch (h->scn) {
              case 2: lrc = launch_cluster<PRE, FMT, ND, 2>(h, chunk, period, s); break;
              case 4: lrc = launch_cluster<PRE, FMT, ND, 4>(h, chunk, period, s); break;
              case 8: lrc = launch_cluster<PRE, FMT, ND, 8>(h, chunk, period, s); break;
              default: lrc = launch_cluster<PRE, FMT, ND, 16>(h, chunk, period, s); break;
            }
            if (lrc) return lrc;
          }
          SG_LAUNCH_CHECK("k_pcg_small");
        }
        return SG_OK;
      });
      if (rc) return rc;
      h->kernels += 1;
      h->chunks += 1;
      it += chunk;
      continue;
    }
    std::vector<int> pattern(chunk);
    for (int c = 0; c < chunk; ++c) pattern[c] = (it + c) > 0 && (it + c) % period == 0;
    cudaGraphExec_t exec;
    rc = get_graph(h, pattern, &exec, &prev_prof);
    if (rc) return rc;
    SG_CUDA(cudaGraphLaunch(exec, s));
    h->kernels += h->graph_kernels[pattern];
    h->chunks += 1;
    it += chunk;
  }
  if (h->D.xdefer && h->nblk > 0) {
    k_xflush<<<(unsigned)h->nblk, PR, 0, s>>>(h->D);
    SG_LAUNCH_CHECK("k_xflush");
    h->kernels += 1;
  }
  if (h->n > 0) SG_CUDA(cudaMemcpyAsync(x, h->D.x, h->n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  SG_CUDA(cudaEventRecord(e1, s));
  SG_CUDA(cudaMemcpyAsync(st.data(), h->st, st.size() * sizeof(SysState), cudaMemcpyDeviceToHost, s));
  SG_CUDA(cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (elapsed_ns_host) *elapsed_ns_host = (int64_t)(ms * 1e6);
  for (int k = 0; k < h->S; ++k) {
    sg_solve_result& R = results_host[k];
    R.k = st[k].i;
    R.converged = st[k].converged;
    R.status = st[k].notspd ? SG_ENOTSPD : SG_OK;
    R.fail_iter = st[k].fail_iter;
    R.fail_value = st[k].fail_value;
    R.fail_kind = st[k].fail_kind;
    R.hist_len = cfg->track_history ? st[k].hist_len : 0;
  }
  return SG_OK;
}

extern "C" int sg_pcg_history(sg_pcg* h, int32_t sys, double* out_host, int64_t len) {
  if (!h || sys < 0 || sys >= h->S) { set_error("bad system index"); return SG_EINVAL; }
  if (len > h->hcap) { set_error("history length exceeds capacity"); return SG_EINVAL; }
  if (len <= 0) return SG_OK;
  SG_CUDA(cudaMemcpy(out_host, h->hist + (long long)sys * h->hcap, len * sizeof(double), cudaMemcpyDeviceToHost));
  return SG_OK;
}

extern "C" int sg_pcg_rebind_values(sg_pcg* h, const double* a_vals, const double* g_vals, const double* gt_vals,
                                    const double* inv_diag) {
  if (!h) { set_error("null handle"); return SG_EINVAL; }
  const bool changed = h->D.a_vals != a_vals || h->D.g_vals != g_vals || h->D.gt_vals != gt_vals ||
                       h->D.inv_diag != inv_diag;
  h->D.a_vals = a_vals;
  h->D.g_vals = g_vals;
  h->D.gt_vals = gt_vals;
  h->D.inv_diag = inv_diag;
  // DIA graphs only read handle-owned arrays (refilled at every solve); CSR graphs captured the
  // value pointers and must be re-captured
  if (changed && !h->dia_nd) {
    for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
    h->graphs.clear();
    h->graph_kernels.clear();
  }
  return SG_OK;
}

extern "C" int sg_pcg_rebind(sg_pcg* h, const int32_t* a_offs, const int32_t* a_cols, const double* a_vals,
                             const int32_t* g_offs, const int32_t* g_cols, const double* g_vals,
                             const int32_t* gt_offs, const int32_t* gt_cols, const double* gt_vals,
                             const double* inv_diag) {
  if (!h) { set_error("null handle"); return SG_EINVAL; }
  Dev& D = h->D;
  const bool moved = D.a_offs != a_offs || D.a_cols != a_cols || D.g_offs != g_offs || D.g_cols != g_cols ||
                     D.gt_offs != gt_offs || D.gt_cols != gt_cols;
  if (moved && h->part) {
    set_error("a row-partitioned PCG handle cannot be re-pointed at other index arrays");
    return SG_EINVAL;
  }
  D.a_offs = a_offs; D.a_cols = a_cols;
  D.g_offs = g_offs; D.g_cols = g_cols;
  D.gt_offs = gt_offs; D.gt_cols = gt_cols;
  if (moved && !h->dia_nd) {  // CSR graphs captured the index pointers
    for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
    h->graphs.clear();
    h->graph_kernels.clear();
  }
  // the next solve fingerprints the patterns behind the new pointers and re-plans if they differ
  return sg_pcg_rebind_values(h, a_vals, g_vals, gt_vals, inv_diag);
}

extern "C" int sg_pcg_set_stencil(sg_pcg* h, const double* coeff, int64_t nx, int64_t ny, int32_t* usable_host) {
  if (!h) { set_error("null handle"); return SG_EINVAL; }
  if (usable_host) *usable_host = 0;
  const Dia& dd = h->D.dia;
  // only the streamed K1 kernels (k_iter1_sw, the strip k_iter1_s5) regenerate A: one-CTA small
  // systems, the tile kernels and the row partition keep the stored diagonals (no per-solve copy +
  // check for them)
  const bool fits = coeff && nx > 1 && ny >= 1 && h->dia_nd == 5 && !h->part &&
                    ((h->staged && h->k1sw && !h->small) || h->strip) &&
                    dd.off[1] == -1 && dd.off[2] == 0 && dd.off[3] == 1 && dd.off[4] == -dd.off[0] &&
                    (int64_t)dd.off[4] == nx;
  const double ihx2 = (double)((nx + 1) * (nx + 1)), ihy2 = (double)((ny + 1) * (ny + 1));  // datasets.py:109-110
  if (fits && h->coef && h->D.ihx2 == ihx2 && h->D.ihy2 == ihy2) {  // only the source array moves
    h->coef_user = coeff;
    if (usable_host) *usable_host = 1;
    return SG_OK;
  }
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);  // the captured Dev changes
  h->graphs.clear();
  h->graph_kernels.clear();
  if (!fits) {
    if (h->coef) cudaFree(h->coef - h->guard);
    h->coef = nullptr;
    h->coef_user = nullptr;
    h->D.coef = nullptr;
    h->cst = 0;
    return SG_OK;
  }
  if (!h->coef) {
    double* base = nullptr;
    SG_CUDA(cudaMalloc(&base, (size_t)(h->n + 2 * h->guard) * sizeof(double)));
    SG_CUDA(cudaMemset(base, 0, (size_t)(h->n + 2 * h->guard) * sizeof(double)));
    h->coef = base + h->guard;
  }
  h->coef_user = coeff;
  h->st_nx = nx;
  h->st_ny = ny;
  h->D.coef = h->coef;
  h->D.ihx2 = ihx2;
  h->D.ihy2 = ihy2;
  h->cst = 0;  // verified against A at every solve
  if (usable_host) *usable_host = 1;
  return SG_OK;
}

extern "C" int sg_pcg_apply_ns(sg_pcg* h, int64_t* ns_host) {
  if (!h || !ns_host) { set_error("null handle"); return SG_EINVAL; }
  *ns_host = 0;
  if (!h->small) return SG_OK;
  unsigned long long v = 0;
  SG_CUDA(cudaMemcpy(&v, &h->ctl->apply_ns, sizeof(v), cudaMemcpyDeviceToHost));
  *ns_host = (int64_t)v;
  return SG_OK;
}

extern "C" int sg_pcg_rebuilds(sg_pcg* h, int64_t* rebuilds_host) {
  if (!h || !rebuilds_host) { set_error("null handle"); return SG_EINVAL; }
  *rebuilds_host = h->rebuilds;
  return SG_OK;
}

extern "C" int sg_pcg_set_trace(sg_pcg* h, void* buf) {
  if (!h) { set_error("null handle"); return SG_EINVAL; }
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  h->graphs.clear();
  h->graph_kernels.clear();
  h->D.trace = static_cast<unsigned long long*>(buf);
  return SG_OK;
}

extern "C" int sg_pcg_set_profile(sg_pcg* h, int32_t on) {
  if (!h) { set_error("null handle"); return SG_EINVAL; }
  if ((on != 0) != (h->profile != 0)) {
    for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
    h->graphs.clear();
    h->graph_kernels.clear();
  }
  h->profile = on ? 1 : 0;
  return SG_OK;
}

extern "C" int sg_pcg_stats(sg_pcg* h, int64_t* kernels_host, int64_t* chunks_host, double* prof_host,
                            int32_t reset) {
  if (!h) { set_error("null handle"); return SG_EINVAL; }
  if (kernels_host) *kernels_host = h->kernels;
  if (chunks_host) *chunks_host = h->chunks;
  if (prof_host) {
    for (int k = 0; k < 3; ++k) prof_host[k] = h->prof_ms[k];
    prof_host[3] = h->prof_active;
    prof_host[4] = h->prof_samples;
    prof_host[5] = h->dia_nd;
    prof_host[6] = h->a_sym ? (h->cst ? 2.0 : 1.0) : 0.0;
    prof_host[7] = (h->staged || h->strip) && h->pre == SG_PRECOND_LEARNED ? 1.0 : 0.0;
  }
  if (reset) {
    h->kernels = h->chunks = 0;
    h->prof_ms[0] = h->prof_ms[1] = h->prof_ms[2] = 0;
    h->prof_active = h->prof_samples = 0;
  }
  return SG_OK;
}

extern "C" void sg_pcg_destroy(sg_pcg* h) {
  if (!h) return;
  for (int k = 0; k < 4; ++k)
    if (h->ev[k]) cudaEventDestroy(h->ev[k]);
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->pinned_active) cudaFreeHost(h->pinned_active);
  cudaDeviceSynchronize();
  if (h->hist) cudaFree(h->hist);
  if (h->dia_mem) cudaFree(h->dia_mem);
  if (h->gblk_mem) cudaFree(h->gblk_mem);
  for (int k = 0; k < 3; ++k) {
    if (h->sell_mem[k]) cudaFree(h->sell_mem[k]);
    if (h->sell_vals[k]) cudaFree(h->sell_vals[k]);
  }
  if (h->d_flag) cudaFree(h->d_flag);
  for (void* pm : h->peer_maps) cudaIpcCloseMemHandle(pm);
  if (h->part_mem) cudaFree(h->part_mem);
  if (h->red_mem) cudaFree(h->red_mem);
  if (h->coef) cudaFree(h->coef - h->guard);
  if (h->mem) cudaFree(h->mem);
  delete h;
}


// ------------------------------------------------------------------ row partition API
namespace {
// Owned ranges + push tables (+ the group sums and counter) in one allocation.
int part_tables(sg_pcg* h, const std::vector<long long>& own0, const std::vector<long long>& own1,
                const std::vector<long long>& plo, const std::vector<long long>& phi,
                const std::vector<double*>& dlo, const std::vector<double*>& dhi, cudaStream_t s) {
  const int S = h->S;
  Carve c(nullptr);
  c.take<long long>(S); c.take<long long>(S); c.take<long long>(S); c.take<long long>(S);
  c.take<double*>(S); c.take<double*>(S); c.take<double>(2 * S); c.take<unsigned int>(4);
  if (h->part_mem) { cudaFree(h->part_mem); h->part_mem = nullptr; }
  SG_CUDA(cudaMalloc(&h->part_mem, c.off));
  SG_CUDA(cudaMemsetAsync(h->part_mem, 0, c.off, s));
  Carve m(h->part_mem);
  long long* d0 = m.take<long long>(S);
  long long* d1 = m.take<long long>(S);
  long long* dl = m.take<long long>(S);
  long long* dh = m.take<long long>(S);
  double** pl = m.take<double*>(S);
  double** ph = m.take<double*>(S);
  double* gs = m.take<double>(2 * S);
  unsigned int* grp = m.take<unsigned int>(4);
  SG_CUDA(cudaMemcpyAsync(d0, own0.data(), S * sizeof(long long), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(d1, own1.data(), S * sizeof(long long), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(dl, plo.data(), S * sizeof(long long), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(dh, phi.data(), S * sizeof(long long), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(pl, dlo.data(), S * sizeof(double*), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(ph, dhi.data(), S * sizeof(double*), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaStreamSynchronize(s));
  Dev& D = h->D;
  D.own0 = d0; D.own1 = d1; D.plo = dl; D.phi = dh; D.push_lo = pl; D.push_hi = ph;
  D.gsum = gs; D.grp = grp; D.nsys = S;
  return SG_OK;
}

// What the partition mode turns off: one-CTA systems, the deferred x update, the coefficient
// stencil (ghost rows are truncated), the CSR long-row kernels; the captured graphs change.
int part_common(sg_pcg* h) {
  if (!h->dia_nd) {
    set_error("the row partition needs a stencil (diagonal-major) pattern");
    return SG_EUNSUPPORTED;
  }
  h->small = 0;
  h->D.xdefer = 0;
  if (h->coef) { cudaFree(h->coef - h->guard); h->coef = nullptr; }
  h->coef_user = nullptr; h->D.coef = nullptr; h->cst = 0;
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  h->graphs.clear();
  h->graph_kernels.clear();
  return SG_OK;
}

struct PeerInfo {  // sg_pcg_peer_info_size() bytes, exchanged between ranks as an opaque blob
  cudaIpcMemHandle_t mem;  // the handle's workspace (vectors)
  cudaIpcMemHandle_t red;  // its reduction block
  int64_t s_off;           // byte offset of s (row 0) inside the workspace
  int64_t n_ext, own_lo, own_hi;
  int32_t world, pad;
};
}  // namespace

extern "C" int sg_pcg_set_partition(sg_pcg* h, const int64_t* own_lo_host, const int64_t* own_hi_host) {
  if (!h || !own_lo_host || !own_hi_host) { set_error("null argument"); return SG_EINVAL; }
  const int S = h->S;
  std::vector<long long> o0(S), o1(S), pl(S, 0), ph(S, 0);
  std::vector<double*> dl(S, nullptr), dh(S, nullptr);
  for (int p = 0; p < S; ++p) {
    const long long n_p = h->sys_start[p + 1] - h->sys_start[p];
    if (!(0 <= own_lo_host[p] && own_lo_host[p] < own_hi_host[p] && own_hi_host[p] <= n_p)) {
      set_error("partition %d: owned rows [%lld, %lld) do not fit its %lld rows", p, (long long)own_lo_host[p],
                (long long)own_hi_host[p], n_p);
      return SG_EINVAL;
    }
    o0[p] = h->sys_start[p] + own_lo_host[p];
    o1[p] = h->sys_start[p] + own_hi_host[p];
  }
  for (int p = 0; p < S; ++p) {  // neighbours are the adjacent systems of the handle
    const long long own = o1[p] - o0[p];
    if (p > 0) {
      pl[p] = h->sys_start[p] - o1[p - 1];  // partition p-1's top ghost rows
      dl[p] = h->D.s + o1[p - 1];
    }
    if (p < S - 1) {
      ph[p] = o0[p + 1] - h->sys_start[p + 1];  // partition p+1's bottom ghost rows
      dh[p] = h->D.s + h->sys_start[p + 1];
    }
    if (pl[p] > own || ph[p] > own) {
      set_error("partition %d owns %lld rows, fewer than its neighbours' ghost depth", p, own);
      return SG_EINVAL;
    }
    if (pl[p] == 0) dl[p] = nullptr;
    if (ph[p] == 0) dh[p] = nullptr;
  }
  int rc = part_common(h);
  if (rc) return rc;
  rc = part_tables(h, o0, o1, pl, ph, dl, dh, nullptr);
  if (rc) return rc;
  h->part_n = 0;
  for (int p = 0; p < S; ++p) h->part_n += o1[p] - o0[p];
  h->part = 1;
  h->D.part = 1;
  return SG_OK;
}

extern "C" int sg_pcg_peer_info_size(void) { return (int)sizeof(PeerInfo); }

extern "C" int sg_pcg_peer_export(sg_pcg* h, int64_t own_lo, int64_t own_hi, int32_t world, void* info_out) {
  if (!h || !info_out) { set_error("null argument"); return SG_EINVAL; }
  if (h->S != 1) { set_error("peer mode: one partition (system) per rank"); return SG_EINVAL; }
  if (world < 1 || world > 8) { set_error("peer mode supports 1..8 ranks"); return SG_EUNSUPPORTED; }
  if (!(0 <= own_lo && own_lo < own_hi && own_hi <= h->n)) { set_error("bad owned row range"); return SG_EINVAL; }
  if (h->red_mem) { cudaFree(h->red_mem); h->red_mem = nullptr; }
  const size_t bytes = (size_t)4 * world * sizeof(double) + (size_t)world * sizeof(unsigned int) + 64;
  SG_CUDA(cudaMalloc(&h->red_mem, bytes));
  SG_CUDA(cudaMemset(h->red_mem, 0, bytes));
  h->red_world = world;
  PeerInfo info{};
  SG_CUDA(cudaIpcGetMemHandle(&info.mem, h->mem));
  SG_CUDA(cudaIpcGetMemHandle(&info.red, h->red_mem));
  info.s_off = (int64_t)(reinterpret_cast<char*>(h->D.s) - static_cast<char*>(h->mem));
  info.n_ext = h->n;
  info.own_lo = own_lo;
  info.own_hi = own_hi;
  info.world = world;
  memcpy(info_out, &info, sizeof(info));
  return SG_OK;
}

extern "C" int sg_pcg_set_peers(sg_pcg* h, int32_t rank, int32_t world, const void* infos) {
  if (!h || !infos) { set_error("null argument"); return SG_EINVAL; }
  if (!h->red_mem || h->red_world != world) { set_error("call sg_pcg_peer_export with this world size first"); return SG_EINVAL; }
  if (rank < 0 || rank >= world) { set_error("bad rank"); return SG_EINVAL; }
  std::vector<PeerInfo> in(world);
  memcpy(in.data(), infos, sizeof(PeerInfo) * world);
  std::vector<char*> mem(world, nullptr), red(world, nullptr);
  for (int q = 0; q < world; ++q) {
    if (in[q].world != world) { set_error("peer %d exported for another world size", q); return SG_EINVAL; }
    if (q == rank) {
      mem[q] = static_cast<char*>(h->mem);
      red[q] = static_cast<char*>(h->red_mem);
      continue;
    }
    void* r = nullptr;
    SG_CUDA(cudaIpcOpenMemHandle(&r, in[q].red, cudaIpcMemLazyEnablePeerAccess));
    h->peer_maps.push_back(r);
    red[q] = static_cast<char*>(r);
    if (q == rank - 1 || q == rank + 1) {
      void* mp = nullptr;
      SG_CUDA(cudaIpcOpenMemHandle(&mp, in[q].mem, cudaIpcMemLazyEnablePeerAccess));
      h->peer_maps.push_back(mp);
      mem[q] = static_cast<char*>(mp);
    }
  }
  const PeerInfo& me = in[rank];
  std::vector<long long> o0{me.own_lo}, o1{me.own_hi}, pl{0}, ph{0};
  std::vector<double*> dl{nullptr}, dh{nullptr};
  const long long own = me.own_hi - me.own_lo;
  if (rank > 0) {  // my first owned rows -> the left neighbour's top ghost rows
    const PeerInfo& L = in[rank - 1];
    pl[0] = L.n_ext - L.own_hi;
    dl[0] = reinterpret_cast<double*>(mem[rank - 1] + L.s_off) + L.own_hi;
  }
  if (rank < world - 1) {  // my last owned rows -> the right neighbour's bottom ghost rows
    const PeerInfo& R = in[rank + 1];
    ph[0] = R.own_lo;
    dh[0] = reinterpret_cast<double*>(mem[rank + 1] + R.s_off);
  }
  if (pl[0] > own || ph[0] > own) { set_error("rank %d owns fewer rows than its neighbours' ghost depth", rank); return SG_EINVAL; }
  if (pl[0] == 0) dl[0] = nullptr;
  if (ph[0] == 0) dh[0] = nullptr;
  int rc = part_common(h);
  if (rc) return rc;
  rc = part_tables(h, o0, o1, pl, ph, dl, dh, nullptr);
  if (rc) return rc;
  Dev& D = h->D;
  D.rank = rank;
  D.nranks = world;
  const size_t gbytes = (size_t)4 * world * sizeof(double);
  for (int q = 0; q < world; ++q) {
    D.peer_gsum[q] = reinterpret_cast<double*>(red[q]);
    D.peer_flag[q] = reinterpret_cast<unsigned int*>(red[q] + gbytes);
  }
  D.gsum = D.peer_gsum[rank];
  D.epoch = reinterpret_cast<unsigned int*>(static_cast<char*>(h->red_mem) + gbytes + world * sizeof(unsigned int));
  h->part_n = 0;
  for (int q = 0; q < world; ++q) h->part_n += in[q].own_hi - in[q].own_lo;
  h->part = 2;
  D.part = 2;
  return SG_OK;
}
