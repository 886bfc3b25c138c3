// Batched, device-resident PCG (pcg.py:131-233).
//
// A batch of independent SPD systems is stored block-diagonally (global column indices).  CTAs
// own ROWS consecutive rows of ONE system, so every dot product is a per-system sum of per-CTA
// partials, reduced deterministically (fixed-shape trees) by the last CTA of that system to
// arrive ("last block" finalizer).  The finalizer runs the reference's scalar control flow
// (alpha, beta, NotSpd checks, refresh, the fresh-residual re-check, max_iters, delta test,
// history) on device, so a system that stops simply makes its CTAs exit early in later
// launches.  The host only launches CUDA graphs of C iterations and polls one counter.
//
// One iteration = three fused kernels (four + two extra on refresh iterations):
//   K1  d' = s + beta d (on the fly for neighbours), q = A d', partial d'.q
//       [+ r_fresh = b - A x and ||r_fresh||^2 when a fresh check / certification is pending]
//   K2  x += alpha d', r' = r - alpha q (on the fly), t = G^T r', partial ||r'||^2
//   K3  s = G t + eps r' (or r' / r' * inv_diag), partial r'.s, finalizer
// Refresh iterations (i > 0, i % period == 0) replace K2 by: x += alpha d'; r' = b - A x;
// t = G^T r'.  Every vector update uses the reference's roundings (no FMA), every SpMV the
// reference's summation order, so the only arithmetic difference from numpy is the order of
// the dot-product reductions (numpy uses OpenBLAS ddot).
#include <map>
#include <vector>

#include "spmv.cuh"

namespace sg {

constexpr int PR = 256;    // rows per CTA (= threads per CTA)
constexpr int PCAP = 2048; // staged nonzeros per CTA (8 per row on average)

enum { ST_RUN = 0, ST_CERTIFY = 1, ST_DONE = 2 };
enum { FL_FRESH = 1 };

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
};

__global__ void k_snapshot(Ctl* c) { c->snap = c->n_active; }

__global__ void k_max_row(const int32_t* __restrict__ offs, int64_t n, unsigned int* out) {
  unsigned int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned int)(offs[i + 1] - offs[i]));
  atomicMax(out, m);
}

struct Dev {
  // block table
  const long long* blk_r0;
  const int* blk_sys;
  const int* sys_blk0;
  // matrices
  const int32_t *a_offs, *a_cols; const double* a_vals;
  const int32_t *g_offs, *g_cols; const double* g_vals;
  const int32_t *gt_offs, *gt_cols; const double* gt_vals;
  const double* inv_diag;
  const long long* sys_r1;  // per system end row
  // vectors
  double *b, *x, *r0, *r1, *d0, *d1, *q, *s, *t;
  // reduction scratch
  double* part;             // [nblk][2]
  unsigned int* counter;    // [S]
  SysState* st;
  Ctl* ctl;
};

__device__ __forceinline__ void block_rows(const Dev& D, int& sys, long long& r0, long long& r1) {
  sys = D.blk_sys[blockIdx.x];
  r0 = D.blk_r0[blockIdx.x];
  const long long e = r0 + PR;
  const long long se = D.sys_r1[sys];
  r1 = e < se ? e : se;
}

// Publish this CTA's two partials; returns true in ALL threads of the last CTA of `sys`.
__device__ __forceinline__ bool arrive(const Dev& D, int sys, double p0, double p1,
                                       double* red, int* flag) {
  double a = block_sum(p0, red);
  double b = block_sum(p1, red);
  if (threadIdx.x == 0) {
    D.part[2 * blockIdx.x + 0] = a;
    D.part[2 * blockIdx.x + 1] = b;
    __threadfence();
    const unsigned int nb = (unsigned)(D.sys_blk0[sys + 1] - D.sys_blk0[sys]);
    const unsigned int old = atomicAdd(&D.counter[sys], 1u);
    *flag = (old == nb - 1);
  }
  __syncthreads();
  const bool last = *flag;
  if (last) __threadfence();
  return last;
}

// Deterministic per-system sum of partial slot `which` (valid in thread 0).
__device__ __forceinline__ double gather_partials(const Dev& D, int sys, int which, double* red) {
  const int b0 = D.sys_blk0[sys], b1 = D.sys_blk0[sys + 1];
  double v = 0.0;
  for (int b = b0 + threadIdx.x; b < b1; b += blockDim.x) v += __ldcg(&D.part[2 * b + which]);
  return block_sum(v, red);
}

__device__ __forceinline__ void finish(const Dev& D, SysState& S, int conv) {
  S.converged = conv;
  S.status = ST_DONE;
  atomicSub(&D.ctl->n_active, 1u);
}

__device__ __forceinline__ void put_hist(const Dev& D, int sys, long long i, double v) {
  const Ctl& c = *D.ctl;
  if (c.track && i < c.hcap) c.hist[(long long)sys * c.hcap + i] = v;
}

// ------------------------------------------------------------------ setup
// r = b; t = G^T b; partial ||b||^2
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_setup1(Dev D) {
  __shared__ RowTile<PR, PCAP> T;
  __shared__ double red[PR / 32];
  __shared__ int flag;
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (PRE == SG_PRECOND_LEARNED) stage_rows(T, r0, r1, D.gt_offs, D.gt_cols, D.gt_vals);
  const long long i = r0 + threadIdx.x;
  double pbb = 0.0;
  if (i < r1) {
    const double bi = D.b[i];
    D.r0[i] = bi;
    D.d0[i] = 0.0;
    D.d1[i] = 0.0;
    D.x[i] = 0.0;
    pbb = mul(bi, bi);
    if (PRE == SG_PRECOND_LEARNED)
      D.t[i] = tile_row_dot<kOrderSeq, SH, 0>(T, threadIdx.x, D.gt_cols, D.gt_vals, XF{D.b, nullptr, 0.0});
  }
  if (arrive(D, sys, pbb, 0.0, red, &flag)) {
    const double bb = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) {
      SysState& S = D.st[sys];
      S.norm_b = __dsqrt_rn(bb);
      S.rr = bb;
      D.counter[sys] = 0;
    }
  }
}

template <int PRE, bool SH>
__device__ __forceinline__ double apply_row(const Dev& D, const RowTile<PR, PCAP>& T, int lr,
                                            long long i, const double* r, double eps) {
  if (PRE == SG_PRECOND_IDENTITY) return r[i];
  if (PRE == SG_PRECOND_JACOBI) return mul(r[i], D.inv_diag[i]);
  const double y = tile_row_dot<kOrderNumpy, SH, 0>(T, lr, D.g_cols, D.g_vals, XF{D.t, nullptr, 0.0});
  return add(y, mul(eps, r[i]));
}

// s = M r0; delta0 = r.s; NotSpd check; top-of-loop checks for i = 0.
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_setup2(Dev D) {
  __shared__ RowTile<PR, PCAP> T;
  __shared__ double red[PR / 32];
  __shared__ int flag;
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (PRE == SG_PRECOND_LEARNED) stage_rows(T, r0, r1, D.g_offs, D.g_cols, D.g_vals);
  const long long i = r0 + threadIdx.x;
  double prs = 0.0;
  if (i < r1) {
    const double si = apply_row<PRE, SH>(D, T, threadIdx.x, i, D.r0, D.ctl->eps);
    D.s[i] = si;
    prs = mul(D.r0[i], si);
  }
  if (arrive(D, sys, prs, 0.0, red, &flag)) {
    const double rs = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) {
      SysState& S = D.st[sys];
      D.counter[sys] = 0;
      const Ctl& c = *D.ctl;
      S.i = 0;
      S.beta = 0.0;
      S.flags = 0;
      S.notspd = 0;
      S.converged = 0;
      if (S.norm_b == 0.0) {  // pcg.py:159-164
        S.hist_len = 1;
        put_hist(D, sys, 0, 0.0);
        finish(D, S, 1);
        return;
      }
      S.hist_len = 1;
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
  }
}

// ------------------------------------------------------------------ K1
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_iter1(Dev D, int par) {
  __shared__ RowTile<PR, PCAP> T;
  __shared__ double red[PR / 32];
  __shared__ int flag;
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  const int status = D.st[sys].status;
  if (status == ST_DONE) return;
  const bool run = status == ST_RUN;
  const bool fresh = run ? (D.st[sys].flags & FL_FRESH) != 0 : true;
  const double beta = D.st[sys].beta;
  double* dc = par ? D.d1 : D.d0;
  double* dn = par ? D.d0 : D.d1;
  double* rc = par ? D.r1 : D.r0;
  stage_rows(T, r0, r1, D.a_offs, D.a_cols, D.a_vals);
  const long long i = r0 + threadIdx.x;
  double pdq = 0.0, prr = 0.0;
  if (i < r1) {
    if (run) {
      const double dni = add(D.s[i], mul(beta, dc[i]));
      dn[i] = dni;
      const double qi = tile_row_dot<kOrderNumpy, SH, 1>(T, threadIdx.x, D.a_cols, D.a_vals, XF{D.s, dc, beta});
      D.q[i] = qi;
      pdq = mul(dni, qi);
    }
    if (fresh) {
      const double ax = tile_row_dot<kOrderNumpy, SH, 0>(T, threadIdx.x, D.a_cols, D.a_vals, XF{D.x, nullptr, 0.0});
      const double rf = sub(D.b[i], ax);
      if (run) rc[i] = rf;
      prr = mul(rf, rf);
    }
  }
  if (arrive(D, sys, pdq, prr, red, &flag)) {
    const double dq = gather_partials(D, sys, 0, red);
    const double rrf = gather_partials(D, sys, 1, red);
    if (threadIdx.x == 0) {
      SysState& S = D.st[sys];
      D.counter[sys] = 0;
      const Ctl& c = *D.ctl;
      if (!run) {  // delta-test certification (pcg.py:217-220)
        const double rel = __ddiv_rn(__dsqrt_rn(rrf), S.norm_b);
        finish(D, S, rel <= c.rtol);
        return;
      }
      if (S.flags & FL_FRESH) {  // pcg.py:208-215
        S.flags &= ~FL_FRESH;
        const double rel = __ddiv_rn(__dsqrt_rn(rrf), S.norm_b);
        put_hist(D, sys, S.i, rel);
        if (rel <= c.rtol) { finish(D, S, 1); return; }
        if (S.i >= S.max_iters) { finish(D, S, 0); return; }
      }
      if (dq <= 0.0) {  // pcg.py:182-184
        S.notspd = 1; S.fail_iter = S.i; S.fail_value = dq; S.fail_kind = 1;
        finish(D, S, 0);
        return;
      }
      S.dq = dq;
      S.alpha = __ddiv_rn(S.delta, dq);
    }
  }
}

// ------------------------------------------------------------------ K2 (non-refresh)
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_iter2(Dev D, int par) {
  __shared__ RowTile<PR, PCAP> T;
  __shared__ double red[PR / 32];
  __shared__ int flag;
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  const double alpha = D.st[sys].alpha;
  const double* dn = par ? D.d0 : D.d1;
  const double* rc = par ? D.r1 : D.r0;
  double* rn = par ? D.r0 : D.r1;
  if (PRE == SG_PRECOND_LEARNED) stage_rows(T, r0, r1, D.gt_offs, D.gt_cols, D.gt_vals);
  const long long i = r0 + threadIdx.x;
  double prr = 0.0;
  if (i < r1) {
    D.x[i] = add(D.x[i], mul(alpha, dn[i]));
    const double rni = sub(rc[i], mul(alpha, D.q[i]));
    rn[i] = rni;
    prr = mul(rni, rni);
    if (PRE == SG_PRECOND_LEARNED)
      D.t[i] = tile_row_dot<kOrderSeq, SH, 2>(T, threadIdx.x, D.gt_cols, D.gt_vals, XF{rc, D.q, alpha});
  }
  if (arrive(D, sys, prr, 0.0, red, &flag)) {
    const double rr = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) {
      D.st[sys].rr = rr;
      D.counter[sys] = 0;
    }
  }
}

// ------------------------------------------------------------------ K2 refresh variants
__global__ void __launch_bounds__(PR) k_refresh_x(Dev D, int par) {
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  const double alpha = D.st[sys].alpha;
  const double* dn = par ? D.d0 : D.d1;
  const long long i = r0 + threadIdx.x;
  if (i < r1) D.x[i] = add(D.x[i], mul(alpha, dn[i]));
}

template <bool SH>
__global__ void __launch_bounds__(PR) k_refresh_r(Dev D, int par) {
  __shared__ RowTile<PR, PCAP> T;
  __shared__ double red[PR / 32];
  __shared__ int flag;
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  double* rn = par ? D.r0 : D.r1;
  stage_rows(T, r0, r1, D.a_offs, D.a_cols, D.a_vals);
  const long long i = r0 + threadIdx.x;
  double prr = 0.0;
  if (i < r1) {
    const double ax = tile_row_dot<kOrderNumpy, SH, 0>(T, threadIdx.x, D.a_cols, D.a_vals, XF{D.x, nullptr, 0.0});
    const double rni = sub(D.b[i], ax);
    rn[i] = rni;
    prr = mul(rni, rni);
  }
  if (arrive(D, sys, prr, 0.0, red, &flag)) {
    const double rr = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) {
      D.st[sys].rr = rr;
      D.counter[sys] = 0;
    }
  }
}

template <bool SH>
__global__ void __launch_bounds__(PR) k_refresh_t(Dev D, int par) {
  __shared__ RowTile<PR, PCAP> T;
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  const double* rn = par ? D.r0 : D.r1;
  stage_rows(T, r0, r1, D.gt_offs, D.gt_cols, D.gt_vals);
  const long long i = r0 + threadIdx.x;
  if (i < r1)
    D.t[i] = tile_row_dot<kOrderSeq, SH, 0>(T, threadIdx.x, D.gt_cols, D.gt_vals, XF{rn, nullptr, 0.0});
}

// ------------------------------------------------------------------ K3
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_iter3(Dev D, int par, int refreshed) {
  __shared__ RowTile<PR, PCAP> T;
  __shared__ double red[PR / 32];
  __shared__ int flag;
  int sys; long long r0, r1;
  block_rows(D, sys, r0, r1);
  if (D.st[sys].status != ST_RUN) return;
  const double* rn = par ? D.r0 : D.r1;
  if (PRE == SG_PRECOND_LEARNED) stage_rows(T, r0, r1, D.g_offs, D.g_cols, D.g_vals);
  const long long i = r0 + threadIdx.x;
  double prs = 0.0;
  if (i < r1) {
    const double si = apply_row<PRE, SH>(D, T, threadIdx.x, i, rn, D.ctl->eps);
    D.s[i] = si;
    prs = mul(rn[i], si);
  }
  if (arrive(D, sys, prs, 0.0, red, &flag)) {
    const double rs = gather_partials(D, sys, 0, red);
    if (threadIdx.x == 0) {
      SysState& S = D.st[sys];
      D.counter[sys] = 0;
      const Ctl& c = *D.ctl;
      const double delta_old = S.delta;
      S.delta = rs;
      if (rs < 0.0) {  // pcg.py:196-198
        S.notspd = 1; S.fail_iter = S.i; S.fail_value = rs; S.fail_kind = 2;
        finish(D, S, 0);
        return;
      }
      S.beta = __ddiv_rn(rs, delta_old);
      S.i += 1;
      const double rel = __ddiv_rn(__dsqrt_rn(S.rr), S.norm_b);
      put_hist(D, sys, S.i, rel);
      S.hist_len = S.i + 1;
      if (!c.delta_mode) {
        if (rel <= c.rtol) {
          if (refreshed) { finish(D, S, 1); return; }
          S.flags |= FL_FRESH;
        } else if (S.i >= S.max_iters) {
          finish(D, S, 0);
        }
      } else if (S.i >= S.max_iters || rs <= S.rtol2d0) {
        S.status = ST_CERTIFY;
      }
    }
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
  // instrumentation: kernel launches, and (when profiling) event nodes around the kernels of
  // one non-refresh iteration per chunk -> per-kernel device time sampled inside the solve
  int64_t kernels = 0, chunks = 0;
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

// Launches one iteration; returns the number of kernels launched through *nk.  With `ev`
// (profiling), external event-record nodes bracket K1, K2 and K3.
// (preconditioner kind) x (SHORT: every row of A, G, G^T has <= 8 entries)
template <class F>
int dispatch(const sg_pcg* h, F f) {
  return dispatch_pre(h->pre, [&](auto P) -> int {
    if (h->short_rows) return f(P, std::integral_constant<bool, true>());
    return f(P, std::integral_constant<bool, false>());
  });
}

int launch_iteration(sg_pcg* h, cudaStream_t s, int par, bool refresh, cudaEvent_t* ev, int* nk) {
  return dispatch(h, [&](auto P, auto SHc) -> int {
    constexpr int PRE = decltype(P)::value;
    constexpr bool SH = decltype(SHc)::value;
    const unsigned g = (unsigned)h->nblk;
    int k = 0;
    if (ev) {
      k_snapshot<<<1, 1, 0, s>>>(h->ctl); ++k;
      SG_CUDA(cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal));
    }
    k_iter1<PRE, SH><<<g, PR, 0, s>>>(h->D, par); ++k;
    if (ev) SG_CUDA(cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal));
    if (!refresh) {
      k_iter2<PRE, SH><<<g, PR, 0, s>>>(h->D, par); ++k;
    } else {
      k_refresh_x<<<g, PR, 0, s>>>(h->D, par); ++k;
      k_refresh_r<SH><<<g, PR, 0, s>>>(h->D, par); ++k;
      if (PRE == SG_PRECOND_LEARNED) { k_refresh_t<SH><<<g, PR, 0, s>>>(h->D, par); ++k; }
    }
    if (ev) SG_CUDA(cudaEventRecordWithFlags(ev[2], s, cudaEventRecordExternal));
    k_iter3<PRE, SH><<<g, PR, 0, s>>>(h->D, par, refresh ? 1 : 0); ++k;
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
  h->S = n_systems;
  h->pre = precond_kind;
  h->eps = epsilon;
  h->sys_start.assign(sys_row_start_host, sys_row_start_host + n_systems + 1);
  h->n = h->sys_start.back();
  std::vector<long long> blk_r0;
  std::vector<int> blk_sys, sys_blk0;
  std::vector<long long> sys_r1;
  for (int k = 0; k < n_systems; ++k) {
    sys_blk0.push_back((int)blk_r0.size());
    const int64_t a = h->sys_start[k], b = h->sys_start[k + 1];
    if (b <= a) { delete h; set_error("every system needs at least one row"); return SG_EINVAL; }
    for (int64_t r = a; r < b; r += PR) { blk_r0.push_back(r); blk_sys.push_back(k); }
    sys_r1.push_back(b);
  }
  sys_blk0.push_back((int)blk_r0.size());
  h->nblk = (int)blk_r0.size();
  const int64_t n = h->n, S = n_systems, nb = h->nblk > 0 ? h->nblk : 1;
  Carve c(nullptr);
  c.take<long long>(nb); c.take<int>(nb); c.take<int>(S + 1); c.take<long long>(S);
  for (int v = 0; v < 9; ++v) c.take<double>(n + 2);
  c.take<double>(2 * nb); c.take<unsigned int>(S); c.take<SysState>(S); c.take<Ctl>(1);
  int e = cudaMalloc(&h->mem, c.off);
  if (e != cudaSuccess) { delete h; return cuda_fail((cudaError_t)e, "cudaMalloc(pcg workspace)"); }
  Carve m(h->mem);
  long long* d_blk_r0 = m.take<long long>(nb);
  int* d_blk_sys = m.take<int>(nb);
  int* d_sys_blk0 = m.take<int>(S + 1);
  long long* d_sys_r1 = m.take<long long>(S);
  double* vec[9];
  for (int v = 0; v < 9; ++v) vec[v] = m.take<double>(n + 2);
  double* part = m.take<double>(2 * nb);
  unsigned int* counter = m.take<unsigned int>(S);
  h->st = m.take<SysState>(S);
  h->ctl = m.take<Ctl>(1);
  if (h->nblk) {
    SG_CUDA(cudaMemcpyAsync(d_blk_r0, blk_r0.data(), blk_r0.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
    SG_CUDA(cudaMemcpyAsync(d_blk_sys, blk_sys.data(), blk_sys.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  }
  SG_CUDA(cudaMemcpyAsync(d_sys_blk0, sys_blk0.data(), sys_blk0.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemcpyAsync(d_sys_r1, sys_r1.data(), sys_r1.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  SG_CUDA(cudaMemsetAsync(counter, 0, S * sizeof(unsigned int), s));
  Dev& D = h->D;
  D.blk_r0 = d_blk_r0; D.blk_sys = d_blk_sys; D.sys_blk0 = d_sys_blk0; D.sys_r1 = d_sys_r1;
  D.a_offs = a_offs; D.a_cols = a_cols; D.a_vals = a_vals;
  D.g_offs = g_offs; D.g_cols = g_cols; D.g_vals = g_vals;
  D.gt_offs = gt_offs; D.gt_cols = gt_cols; D.gt_vals = gt_vals;
  D.inv_diag = inv_diag;
  D.b = vec[0]; D.x = vec[1]; D.r0 = vec[2]; D.r1 = vec[3]; D.d0 = vec[4]; D.d1 = vec[5];
  D.q = vec[6]; D.s = vec[7]; D.t = vec[8];
  D.part = part; D.counter = counter; D.st = h->st; D.ctl = h->ctl;
  SG_CUDA(cudaHostAlloc(&h->pinned_active, 2 * sizeof(unsigned int), cudaHostAllocDefault));
  SG_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
  for (int k = 0; k < 4; ++k) SG_CUDA(cudaEventCreate(&h->ev[k]));
  {  // longest row of every matrix the loop touches -> SHORT kernels when all are <= 8
    unsigned int* mx = counter;  // reuse (zeroed again below)
    SG_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned int), s));
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
    h->short_rows = hm <= 8 ? 1 : 0;
    SG_CUDA(cudaMemsetAsync(counter, 0, S * sizeof(unsigned int), s));
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
    h->chunk = chunk;
    h->period = period;
  }
  // per-system state
  std::vector<SysState> st(h->S);
  for (int k = 0; k < h->S; ++k) {
    memset(&st[k], 0, sizeof(SysState));
    const int64_t ns = h->sys_start[k + 1] - h->sys_start[k];
    st[k].max_iters = cfg->max_iters < 0 ? 20 * ns : cfg->max_iters;
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
  if (g) {
    rc = dispatch(h, [&](auto P, auto SHc) -> int {
      constexpr int PRE = decltype(P)::value;
      constexpr bool SH = decltype(SHc)::value;
      k_setup1<PRE, SH><<<g, PR, 0, s>>>(h->D);
      k_setup2<PRE, SH><<<g, PR, 0, s>>>(h->D);
      SG_LAUNCH_CHECK("pcg setup");
      return SG_OK;
    });
    if (rc) return rc;
  } else {
    // all systems empty: nothing to iterate (norm_b == 0 path)
    for (int k = 0; k < h->S; ++k) { st[k].status = ST_DONE; st[k].converged = 1; st[k].hist_len = 1; }
    SG_CUDA(cudaMemcpyAsync(h->st, st.data(), st.size() * sizeof(SysState), cudaMemcpyHostToDevice, s));
  }
  // device-resident loop: graphs of `chunk` iterations, poll the active count between chunks
  if (g) h->kernels += 2;
  int64_t it = 0;
  int prev_prof = -1;
  while (g) {
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
    }
    if (h->pinned_active[0] == 0) break;
    if (cfg->track_history) {
      rc = ensure_hist(h, it + chunk + 2, s);
      if (rc) return rc;
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
  if (h->mem) cudaFree(h->mem);
  delete h;
}
