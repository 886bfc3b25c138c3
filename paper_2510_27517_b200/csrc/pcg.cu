// Batched, device-resident PCG (pcg.py:131-233).
//
// A batch of independent SPD systems is stored block-diagonally (global column indices).  Rows
// are cut into TILES of PR rows that never straddle two systems; every dot product is a
// per-system sum of per-tile partials, reduced deterministically (fixed-shape trees) by the CTA
// that completes the system's last tile.  That CTA also runs the reference's scalar control
// flow (alpha, beta, NotSpd checks, refresh, the fresh-residual re-check, max_iters, the delta
// test, history) on device, so a system that stops makes its tiles be skipped afterwards.  The
// host only launches CUDA graphs of one refresh period of iterations and polls one counter.
//
// Kernels are PERSISTENT: gridDim = SMs x resident CTAs, tiles assigned round-robin (so the work
// of every system spreads over all SMs, which keeps the load balanced while systems drop out).
// Each CTA runs a 2-stage pipeline: while it reduces tile k from shared memory, the TMA engine
// (cp.async.bulk + mbarrier) streams the row offsets, values and column indices of its next
// tile into the other buffer.
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
#include <map>
#include <vector>

#include "spmv.cuh"
#include "tma.cuh"

namespace sg {

constexpr int PR = 256;    // rows per tile (= threads per CTA)
constexpr int PCAP = 2048; // staged nonzeros per tile (8 per row on average)

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
  // tile table
  const long long* blk_r0;
  const int* blk_sys;
  const int* sys_blk0;
  const long long* sys_r1;  // per system end row
  int nblk;
  // matrices
  const int32_t *a_offs, *a_cols; const double* a_vals;
  const int32_t *g_offs, *g_cols; const double* g_vals;
  const int32_t *gt_offs, *gt_cols; const double* gt_vals;
  const double* inv_diag;
  // vectors
  double *b, *x, *r0, *r1, *d0, *d1, *q, *s, *t;
  // reduction scratch
  double* part;             // [nblk][2]
  unsigned int* counter;    // [S]
  SysState* st;
  Ctl* ctl;
};

// ------------------------------------------------------------------ tile pipeline
struct __align__(16) Pipe {
  double vals[2][PCAP + 2];
  int32_t cols[2][PCAP + 4];
  int32_t offs[2][PR + 8];
  uint64_t bar[2];
  int meta[2][4];  // base_v, base_c, base_o, staged
  double red[PR / 32];
  int flag;
};

struct Mat {
  const int32_t* offs;
  const int32_t* cols;
  const double* vals;
};

// Issue the bulk copies of tile t into buffer `buf` (one thread).
__device__ __forceinline__ void issue_tile(const Dev& D, Pipe& P, const Mat& M, int t, int buf) {
  const int sys = D.blk_sys[t];
  const long long r0 = D.blk_r0[t];
  const long long r1 = min(r0 + PR, D.sys_r1[sys]);
  const int e0 = __ldg(M.offs + r0), e1 = __ldg(M.offs + r1);
  const int a0v = e0 & ~1, a1v = (e1 + 1) & ~1;
  const int a0c = e0 & ~3, a1c = (e1 + 3) & ~3;
  const long long o0 = r0 & ~3LL, o1 = (r1 + 1 + 3) & ~3LL;
  const bool fits = (a1v - a0v) <= PCAP + 2 && (a1c - a0c) <= PCAP + 4;
  const uint32_t ob = (uint32_t)((o1 - o0) * 4);
  const uint32_t vb = fits ? (uint32_t)((a1v - a0v) * 8) : 0u;
  const uint32_t cb = fits ? (uint32_t)((a1c - a0c) * 4) : 0u;
  P.meta[buf][0] = a0v;
  P.meta[buf][1] = a0c;
  P.meta[buf][2] = (int)o0;
  P.meta[buf][3] = fits ? 1 : 0;
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(&P.bar[buf], ob + vb + cb);
  bulk_g2s(P.offs[buf], M.offs + o0, ob, &P.bar[buf]);
  if (vb) bulk_g2s(P.vals[buf], M.vals + a0v, vb, &P.bar[buf]);
  if (cb) bulk_g2s(P.cols[buf], M.cols + a0c, cb, &P.bar[buf]);
}

// View of one staged tile: pointers valid for global entry / row indices of that tile.
struct TileView {
  const double* v;
  const int32_t* c;
  const int32_t* o;  // o[i] = row offset of global row i
};

__device__ __forceinline__ TileView view(const Pipe& P, const Mat& M, int buf) {
  TileView tv;
  tv.o = P.offs[buf] - P.meta[buf][2];
  if (P.meta[buf][3]) {
    tv.v = P.vals[buf] - P.meta[buf][0];
    tv.c = P.cols[buf] - P.meta[buf][1];
  } else {
    tv.v = M.vals;
    tv.c = M.cols;
  }
  return tv;
}

// Next tile >= t (stride gridDim.x) whose system satisfies `want(status)`; D.nblk if none.
template <class Want>
__device__ __forceinline__ int next_tile(const Dev& D, int t, const Want& want) {
  for (; t < D.nblk; t += gridDim.x)
    if (want(D.st[D.blk_sys[t]].status)) return t;
  return D.nblk;
}

// Round-robin persistent loop over the CTA's tiles with a 2-stage TMA pipeline.
// body(t, sys, r0, r1, TileView) is executed by all threads and must be CTA-uniform.
template <bool STAGE, class Want, class Body>
__device__ __forceinline__ void tile_loop(const Dev& D, Pipe& P, const Mat& M, const Want& want, const Body& body) {
  if (STAGE && threadIdx.x == 0) {
    mbar_init(&P.bar[0], 1);
    mbar_init(&P.bar[1], 1);
    mbar_init_fence();
  }
  __syncthreads();
  int t = next_tile(D, blockIdx.x, want);
  if (STAGE && threadIdx.x == 0 && t < D.nblk) issue_tile(D, P, M, t, 0);
  int buf = 0;
  uint32_t phase0 = 0, phase1 = 0;
  while (t < D.nblk) {
    const int tn = next_tile(D, t + gridDim.x, want);
    if (STAGE && threadIdx.x == 0 && tn < D.nblk) issue_tile(D, P, M, tn, buf ^ 1);
    const int sys = D.blk_sys[t];
    const long long r0 = D.blk_r0[t];
    const long long r1 = min(r0 + PR, D.sys_r1[sys]);
    TileView tv{M.vals, M.cols, M.offs};
    if (STAGE) {
      mbar_wait(&P.bar[buf], buf ? phase1 : phase0);
      if (buf) phase1 ^= 1u; else phase0 ^= 1u;
      tv = view(P, M, buf);
    }
    body(t, sys, r0, r1, tv);
    __syncthreads();  // buffer `buf` is free again; body's shared scratch may be reused
    t = tn;
    buf ^= 1;
  }
}

// Publish tile t's two partials; returns true in ALL threads of the CTA that completed the
// last tile of `sys`.
__device__ __forceinline__ bool arrive(const Dev& D, Pipe& P, int t, int sys, double p0, double p1) {
  const double a = block_sum(p0, P.red);
  const double b = block_sum(p1, P.red);
  if (threadIdx.x == 0) {
    D.part[2 * t + 0] = a;
    D.part[2 * t + 1] = b;
    __threadfence();
    const unsigned int nb = (unsigned)(D.sys_blk0[sys + 1] - D.sys_blk0[sys]);
    const unsigned int old = atomicAdd(&D.counter[sys], 1u);
    P.flag = (old == nb - 1);
  }
  __syncthreads();
  const bool last = P.flag;
  if (last) __threadfence();
  return last;
}

// Deterministic per-system sum of partial slot `which` (valid in thread 0).
__device__ __forceinline__ double gather_partials(const Dev& D, Pipe& P, int sys, int which) {
  const int b0 = D.sys_blk0[sys], b1 = D.sys_blk0[sys + 1];
  double v = 0.0;
  for (int b = b0 + threadIdx.x; b < b1; b += blockDim.x) v += __ldcg(&D.part[2 * b + which]);
  return block_sum(v, P.red);
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

struct WantAll { __device__ bool operator()(int) const { return true; } };
struct WantRun { __device__ bool operator()(int s) const { return s == ST_RUN; } };
struct WantLive { __device__ bool operator()(int s) const { return s != ST_DONE; } };

template <int PRE>
__device__ __forceinline__ Mat mat_g(const Dev& D) { return Mat{D.g_offs, D.g_cols, D.g_vals}; }
__device__ __forceinline__ Mat mat_gt(const Dev& D) { return Mat{D.gt_offs, D.gt_cols, D.gt_vals}; }
__device__ __forceinline__ Mat mat_a(const Dev& D) { return Mat{D.a_offs, D.a_cols, D.a_vals}; }

template <int ORDER, bool SH, int XM>
__device__ __forceinline__ double trow(const TileView& tv, long long i, const XF& f) {
  return row_reduce<ORDER, SH, XM>(tv.v, tv.c, tv.o[i], tv.o[i + 1], f);
}

// ------------------------------------------------------------------ setup
// r = b; d = 0; x = 0; t = G^T b; partial ||b||^2
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_setup1(Dev D) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Pipe& P = *reinterpret_cast<Pipe*>(smem_raw);
  tile_loop<PRE == SG_PRECOND_LEARNED>(D, P, mat_gt(D), WantAll{},
      [&](int t, int sys, long long r0, long long r1, const TileView& tv) {
    const long long i = r0 + threadIdx.x;
    double pbb = 0.0;
    if (i < r1) {
      const double bi = D.b[i];
      D.r0[i] = bi;
      D.d0[i] = 0.0;
      D.d1[i] = 0.0;
      D.x[i] = 0.0;
      pbb = mul(bi, bi);
      if (PRE == SG_PRECOND_LEARNED) D.t[i] = trow<kOrderSeq, SH, 0>(tv, i, XF{D.b, nullptr, 0.0});
    }
    if (arrive(D, P, t, sys, pbb, 0.0)) {
      const double bb = gather_partials(D, P, sys, 0);
      if (threadIdx.x == 0) {
        SysState& S = D.st[sys];
        S.norm_b = __dsqrt_rn(bb);
        S.rr = bb;
        D.counter[sys] = 0;
      }
    }
  });
}

template <int PRE, bool SH>
__device__ __forceinline__ double apply_row(const Dev& D, const TileView& tv, long long i, const double* r,
                                            double eps) {
  if (PRE == SG_PRECOND_IDENTITY) return r[i];
  if (PRE == SG_PRECOND_JACOBI) return mul(r[i], D.inv_diag[i]);
  const double y = trow<kOrderNumpy, SH, 0>(tv, i, XF{D.t, nullptr, 0.0});
  return add(y, mul(eps, r[i]));
}

// s = M r0; delta0 = r.s; NotSpd check; top-of-loop checks for i = 0.
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_setup2(Dev D) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Pipe& P = *reinterpret_cast<Pipe*>(smem_raw);
  const double eps = D.ctl->eps;
  tile_loop<PRE == SG_PRECOND_LEARNED>(D, P, mat_g<PRE>(D), WantAll{},
      [&](int t, int sys, long long r0, long long r1, const TileView& tv) {
    const long long i = r0 + threadIdx.x;
    double prs = 0.0;
    if (i < r1) {
      const double si = apply_row<PRE, SH>(D, tv, i, D.r0, eps);
      D.s[i] = si;
      prs = mul(D.r0[i], si);
    }
    if (arrive(D, P, t, sys, prs, 0.0)) {
      const double rs = gather_partials(D, P, sys, 0);
      if (threadIdx.x == 0) {
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
    }
  });
}

// ------------------------------------------------------------------ K1
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_iter1(Dev D, int par) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Pipe& P = *reinterpret_cast<Pipe*>(smem_raw);
  double* dc = par ? D.d1 : D.d0;
  double* dn = par ? D.d0 : D.d1;
  double* rc = par ? D.r1 : D.r0;
  tile_loop<true>(D, P, mat_a(D), WantLive{},
      [&](int t, int sys, long long r0, long long r1, const TileView& tv) {
    const int status = D.st[sys].status;
    const bool run = status == ST_RUN;
    const bool fresh = run ? (D.st[sys].flags & FL_FRESH) != 0 : true;
    const double beta = D.st[sys].beta;
    const long long i = r0 + threadIdx.x;
    double pdq = 0.0, prr = 0.0;
    if (i < r1) {
      if (run) {
        const double dni = add(D.s[i], mul(beta, dc[i]));
        dn[i] = dni;
        const double qi = trow<kOrderNumpy, SH, 1>(tv, i, XF{D.s, dc, beta});
        D.q[i] = qi;
        pdq = mul(dni, qi);
      }
      if (fresh) {
        const double rf = sub(D.b[i], trow<kOrderNumpy, SH, 0>(tv, i, XF{D.x, nullptr, 0.0}));
        if (run) rc[i] = rf;
        prr = mul(rf, rf);
      }
    }
    if (arrive(D, P, t, sys, pdq, prr)) {
      const double dq = gather_partials(D, P, sys, 0);
      const double rrf = gather_partials(D, P, sys, 1);
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
  });
}

// ------------------------------------------------------------------ K2 (non-refresh)
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_iter2(Dev D, int par) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Pipe& P = *reinterpret_cast<Pipe*>(smem_raw);
  const double* dn = par ? D.d0 : D.d1;
  const double* rc = par ? D.r1 : D.r0;
  double* rn = par ? D.r0 : D.r1;
  tile_loop<PRE == SG_PRECOND_LEARNED>(D, P, mat_gt(D), WantRun{},
      [&](int t, int sys, long long r0, long long r1, const TileView& tv) {
    const double alpha = D.st[sys].alpha;
    const long long i = r0 + threadIdx.x;
    double prr = 0.0;
    if (i < r1) {
      D.x[i] = add(D.x[i], mul(alpha, dn[i]));
      const double rni = sub(rc[i], mul(alpha, D.q[i]));
      rn[i] = rni;
      prr = mul(rni, rni);
      if (PRE == SG_PRECOND_LEARNED) D.t[i] = trow<kOrderSeq, SH, 2>(tv, i, XF{rc, D.q, alpha});
    }
    if (arrive(D, P, t, sys, prr, 0.0)) {
      const double rr = gather_partials(D, P, sys, 0);
      if (threadIdx.x == 0) {
        D.st[sys].rr = rr;
        D.counter[sys] = 0;
      }
    }
  });
}

// ------------------------------------------------------------------ K2 refresh variants
__global__ void __launch_bounds__(PR) k_refresh_x(Dev D, int par) {
  const double* dn = par ? D.d0 : D.d1;
  for (int t = blockIdx.x; t < D.nblk; t += gridDim.x) {
    const int sys = D.blk_sys[t];
    if (D.st[sys].status != ST_RUN) continue;
    const double alpha = D.st[sys].alpha;
    const long long r0 = D.blk_r0[t];
    const long long i = r0 + threadIdx.x;
    if (i < min(r0 + PR, D.sys_r1[sys])) D.x[i] = add(D.x[i], mul(alpha, dn[i]));
  }
}

template <bool SH>
__global__ void __launch_bounds__(PR) k_refresh_r(Dev D, int par) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Pipe& P = *reinterpret_cast<Pipe*>(smem_raw);
  double* rn = par ? D.r0 : D.r1;
  tile_loop<true>(D, P, mat_a(D), WantRun{},
      [&](int t, int sys, long long r0, long long r1, const TileView& tv) {
    const long long i = r0 + threadIdx.x;
    double prr = 0.0;
    if (i < r1) {
      const double rni = sub(D.b[i], trow<kOrderNumpy, SH, 0>(tv, i, XF{D.x, nullptr, 0.0}));
      rn[i] = rni;
      prr = mul(rni, rni);
    }
    if (arrive(D, P, t, sys, prr, 0.0)) {
      const double rr = gather_partials(D, P, sys, 0);
      if (threadIdx.x == 0) {
        D.st[sys].rr = rr;
        D.counter[sys] = 0;
      }
    }
  });
}

template <bool SH>
__global__ void __launch_bounds__(PR) k_refresh_t(Dev D, int par) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Pipe& P = *reinterpret_cast<Pipe*>(smem_raw);
  const double* rn = par ? D.r0 : D.r1;
  tile_loop<true>(D, P, mat_gt(D), WantRun{},
      [&](int t, int sys, long long r0, long long r1, const TileView& tv) {
    const long long i = r0 + threadIdx.x;
    if (i < r1) D.t[i] = trow<kOrderSeq, SH, 0>(tv, i, XF{rn, nullptr, 0.0});
  });
}

// ------------------------------------------------------------------ K3
template <int PRE, bool SH>
__global__ void __launch_bounds__(PR) k_iter3(Dev D, int par, int refreshed) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Pipe& P = *reinterpret_cast<Pipe*>(smem_raw);
  const double* rn = par ? D.r0 : D.r1;
  const double eps = D.ctl->eps;
  tile_loop<PRE == SG_PRECOND_LEARNED>(D, P, mat_g<PRE>(D), WantRun{},
      [&](int t, int sys, long long r0, long long r1, const TileView& tv) {
    const long long i = r0 + threadIdx.x;
    double prs = 0.0;
    if (i < r1) {
      const double si = apply_row<PRE, SH>(D, tv, i, rn, eps);
      D.s[i] = si;
      prs = mul(rn[i], si);
    }
    if (arrive(D, P, t, sys, prs, 0.0)) {
      const double rs = gather_partials(D, P, sys, 0);
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
  });
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
  unsigned grid = 0;  // persistent CTAs per kernel
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

// (preconditioner kind) x (SHORT: every row of A, G, G^T has <= 8 entries)
template <class F>
int dispatch(const sg_pcg* h, F f) {
  return dispatch_pre(h->pre, [&](auto P) -> int {
    if (h->short_rows) return f(P, std::integral_constant<bool, true>());
    return f(P, std::integral_constant<bool, false>());
  });
}

constexpr size_t kSmem = sizeof(Pipe);

// Opt every pipelined kernel of this (PRE, SH) into the dynamic shared memory it needs and
// size the persistent grid from the occupancy of the heaviest one.
int configure(sg_pcg* h) {
  return dispatch(h, [&](auto P, auto SHc) -> int {
    constexpr int PRE = decltype(P)::value;
    constexpr bool SH = decltype(SHc)::value;
    const void* fns[] = {(const void*)k_setup1<PRE, SH>, (const void*)k_setup2<PRE, SH>,
                         (const void*)k_iter1<PRE, SH>, (const void*)k_iter2<PRE, SH>,
                         (const void*)k_iter3<PRE, SH>, (const void*)k_refresh_r<SH>,
                         (const void*)k_refresh_t<SH>};
    int occ = 1 << 30;
    for (const void* f : fns) {
      SG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
      int o = 0;
      SG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, f, PR, kSmem));
      occ = o < occ ? o : occ;
    }
    int dev = 0, sms = 0;
    SG_CUDA(cudaGetDevice(&dev));
    SG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long long g = (long long)sms * (occ > 0 ? occ : 1);
    h->grid = (unsigned)(g < h->nblk ? g : h->nblk);
    if (h->grid == 0) h->grid = 1;
    return SG_OK;
  });
}

// Launches one iteration; returns the number of kernels launched through *nk.  With `ev`
// (profiling), external event-record nodes bracket K1, K2 and K3.
int launch_iteration(sg_pcg* h, cudaStream_t s, int par, bool refresh, cudaEvent_t* ev, int* nk) {
  return dispatch(h, [&](auto P, auto SHc) -> int {
    constexpr int PRE = decltype(P)::value;
    constexpr bool SH = decltype(SHc)::value;
    const unsigned g = h->grid;
    int k = 0;
    if (ev) {
      k_snapshot<<<1, 1, 0, s>>>(h->ctl); ++k;
      SG_CUDA(cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal));
    }
    k_iter1<PRE, SH><<<g, PR, kSmem, s>>>(h->D, par); ++k;
    if (ev) SG_CUDA(cudaEventRecordWithFlags(ev[1], s, cudaEventRecordExternal));
    if (!refresh) {
      k_iter2<PRE, SH><<<g, PR, kSmem, s>>>(h->D, par); ++k;
    } else {
      k_refresh_x<<<g, PR, 0, s>>>(h->D, par); ++k;
      k_refresh_r<SH><<<g, PR, kSmem, s>>>(h->D, par); ++k;
      if (PRE == SG_PRECOND_LEARNED) { k_refresh_t<SH><<<g, PR, kSmem, s>>>(h->D, par); ++k; }
    }
    if (ev) SG_CUDA(cudaEventRecordWithFlags(ev[2], s, cudaEventRecordExternal));
    k_iter3<PRE, SH><<<g, PR, kSmem, s>>>(h->D, par, refresh ? 1 : 0); ++k;
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
  D.nblk = h->nblk;
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
  int rc = configure(h);
  if (rc) return rc;
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
  const unsigned g = h->grid;
  rc = dispatch(h, [&](auto P, auto SHc) -> int {
    constexpr int PRE = decltype(P)::value;
    constexpr bool SH = decltype(SHc)::value;
    k_setup1<PRE, SH><<<g, PR, kSmem, s>>>(h->D);
    k_setup2<PRE, SH><<<g, PR, kSmem, s>>>(h->D);
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
