// GNN forward (gnn.py:208-253) restructured for the GPU, on FP64 tensor
// cores.
//
// With message_uses_hidden_edge = False the node path never reads the edge state H, and the
// first layer of every MLP on a concatenation is linear.  So
//   * node path, per layer t: P = X W1m[0:D], Q = X W1m[D:2D] are node-level products; the
//     message MLP's hidden activations are summed per CSR row, act(P_i + Q_j + e_k c + b1),
//     and its (linear) second layer is applied AFTER the row sum: m = S W2m + deg b2m;
//     X += f_v(m).  One kernel per layer, fused with the node-level products the next stages
//     need (P'_t, Q'_t for the edge pass; P, Q for layer t+1).
//   * edge pass: ONE kernel; h stays in registers through all L layers:
//     h = E_e(e); h += f_e-second-layer(act(P'_t[i] + Q'_t[j] + h W1e[2D:3D] + b1e)); g = D(h).
//     H never touches HBM (the reference tape holds ~18 KB per edge).
//
// Every [rows x D] . [D x D] product runs on the FP64 tensor cores (mma.sync.m8n8k4.f64, DMMA):
// a warp owns 8 rows (8 edges or 8 nodes); lane (r = lane/4, c = lane%4) holds the features
// f = 8*nb + 2*c + s (nb < D/8, s < 2) of row r — exactly the accumulator layout of the MMA.
// Feeding an accumulator back as the next A operand only needs the k dimension permuted, which
// is folded into the weights: the B fragments are pre-arranged in shared memory so that k-step
// kb pairs with the lane's held value v[kb].  Activations, biases and residuals are
// elementwise in that layout, so consecutive matvecs never shuffle data between lanes.
// Node-level arrays are row-major [node][DP] (DP = D padded to 8), so the 4 lanes of a row read
// 64 contiguous bytes per n-tile.  fp64 throughout (parity is tolerance-based).
#include "common.cuh"
#include "tc.cuh"

namespace sg {

template <int ACT>
__device__ __forceinline__ double act_fn(double v) {
  if (ACT == 0) return v > 0.0 ? v : 0.0;
  return tanh(v);
}

struct MlpP {  // one MLP with a single hidden layer: W1 (din x D), b1, W2 (D x dout), b2
  const double *W1, *b1, *W2, *b2;
};

struct GnnP {
  MlpP en, ee, dec;
  MlpP fm[16], fv[16], fe[16];
  int L, dn;
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int D>
struct Shape {
  static constexpr int DP = (D + 7) / 8 * 8;  // padded width
  static constexpr int NB = DP / 8;           // n-tiles (8 outputs each)
  static constexpr int KS = DP / 4;           // k-steps (4 inputs each) == values held per lane
  static constexpr int FRAG = KS * NB * 32;   // doubles per weight matrix in fragment layout
};

// Feature held by lane-column c at value index v (v = 2*nb + s).
__device__ __forceinline__ int feat(int v, int c) { return 8 * (v >> 1) + 2 * c + (v & 1); }

// Stage W (rows row0.. of a row-major [rows x D] matrix, D_in = D used rows) into fragment
// layout: frag[(kb*NB + nb)*32 + lane] = W[row0 + feat(kb, lane%4)][8*nb + lane/4] (0 if padded).
template <int D>
__device__ void stage_frag(double* dst, const double* __restrict__ W, int row0) {
  using S = Shape<D>;
  for (int idx = threadIdx.x; idx < S::FRAG; idx += blockDim.x) {
    const int ln = idx & 31, kbnb = idx >> 5;
    const int kb = kbnb / S::NB, nb = kbnb % S::NB;
    const int k = feat(kb, ln & 3), nn = 8 * nb + (ln >> 2);
    dst[idx] = (k < D && nn < D) ? W[(int64_t)(row0 + k) * D + nn] : 0.0;
  }
}

// Padded vector (bias / single weight row) into shared memory.
template <int D>
__device__ void stage_vec(double* dst, const double* __restrict__ v) {
  for (int f = threadIdx.x; f < Shape<D>::DP; f += blockDim.x) dst[f] = f < D ? v[f] : 0.0;
}

// out (accumulator layout) += in (accumulator layout) . W (fragment layout in shared memory)
template <int D>
__device__ __forceinline__ void mv(const double* in, const double* __restrict__ Wf, double* out, int lane) {
  using S = Shape<D>;
#pragma unroll
  for (int nb = 0; nb < S::NB; ++nb) {
    double d0 = out[2 * nb], d1 = out[2 * nb + 1];
#pragma unroll
    for (int kb = 0; kb < S::KS; ++kb) dmma(d0, d1, in[kb], Wf[(kb * S::NB + nb) * 32 + lane]);
    out[2 * nb] = d0;
    out[2 * nb + 1] = d1;
  }
}

// Row-major padded row access for the lane's values: row[v] for v = 2nb + s -> row + feat.
__device__ __forceinline__ void load_row(double* v, const double* __restrict__ row, int c, int KS) {
  for (int nb = 0; nb < KS / 2; ++nb) {
    const double2 p = *reinterpret_cast<const double2*>(row + 8 * nb + 2 * c);
    v[2 * nb] = p.x;
    v[2 * nb + 1] = p.y;
  }
}

// ------------------------------------------------------------------ node encoder
// X = E_n(V); PQ = [X W1m0[0:D] | X W1m0[D:2D]] (layer 0's node products), rows padded to DP.
template <int D, int ACT>
__global__ void __launch_bounds__(128) k_node_encode(GnnP p, int64_t n, const double* __restrict__ V,
                                                     double* __restrict__ X, double* __restrict__ PQ) {
  using S = Shape<D>;
  constexpr int DP = S::DP, KS = S::KS;
  extern __shared__ __align__(16) double sm[];
  double* W1 = sm;                     // [4][DP] rows of E_n's first layer (d_node <= 4)
  double* b1 = W1 + 4 * DP;
  double* b2 = b1 + DP;
  double* F2 = b2 + DP;                // E_n second layer
  double* FP = F2 + S::FRAG;           // layer-0 P weights
  double* FQ = FP + S::FRAG;           // layer-0 Q weights
  for (int k = 0; k < 4; ++k)
    for (int f = threadIdx.x; f < DP; f += blockDim.x)
      W1[k * DP + f] = (k < p.dn && f < D) ? p.en.W1[k * D + f] : 0.0;
  stage_vec<D>(b1, p.en.b1);
  stage_vec<D>(b2, p.en.b2);
  stage_frag<D>(F2, p.en.W2, 0);
  if (p.L > 0) {
    stage_frag<D>(FP, p.fm[0].W1, 0);
    stage_frag<D>(FQ, p.fm[0].W1, D);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t base = (int64_t)(blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 8; base < n; base += warps * 8) {
    const int64_t i = base + r;
    const bool ok = i < n;
    double h[KS], x[KS];
#pragma unroll
    for (int v = 0; v < KS; ++v) {
      const int f = feat(v, c);
      double a = b1[f];
      for (int k = 0; k < p.dn; ++k) a = fma(ok ? V[i * p.dn + k] : 0.0, W1[k * DP + f], a);
      h[v] = act_fn<ACT>(a);
      x[v] = b2[f];
    }
    mv<D>(h, F2, x, lane);
    if (ok) {
#pragma unroll
      for (int nb = 0; nb < KS / 2; ++nb)
        *reinterpret_cast<double2*>(X + i * DP + 8 * nb + 2 * c) = make_double2(x[2 * nb], x[2 * nb + 1]);
    }
    if (p.L > 0) {
      double q[KS];
#pragma unroll
      for (int v = 0; v < KS; ++v) q[v] = 0.0;
      mv<D>(x, FP, q, lane);
      if (ok) {
#pragma unroll
        for (int nb = 0; nb < KS / 2; ++nb)
          *reinterpret_cast<double2*>(PQ + i * 2 * DP + 8 * nb + 2 * c) = make_double2(q[2 * nb], q[2 * nb + 1]);
      }
#pragma unroll
      for (int v = 0; v < KS; ++v) q[v] = 0.0;
      mv<D>(x, FQ, q, lane);
      if (ok) {
#pragma unroll
        for (int nb = 0; nb < KS / 2; ++nb)
          *reinterpret_cast<double2*>(PQ + i * 2 * DP + DP + 8 * nb + 2 * c) = make_double2(q[2 * nb], q[2 * nb + 1]);
      }
    }
  }
}

// ------------------------------------------------------------------ node layer t
template <int D>
__host__ __device__ constexpr int node_layer_smem_doubles() {
  return 7 * Shape<D>::FRAG + 6 * Shape<D>::DP;
}

template <int D, int ACT>
__global__ void __launch_bounds__(128) k_node_layer(GnnP p, int t, int64_t n, const int32_t* __restrict__ offs,
                                                    const int32_t* __restrict__ cols,
                                                    const double* __restrict__ ef, double* __restrict__ X,
                                                    const double* __restrict__ PQ, double* __restrict__ PQn,
                                                    double* __restrict__ EPQ) {
  using S = Shape<D>;
  constexpr int DP = S::DP, KS = S::KS, F = S::FRAG;
  extern __shared__ __align__(16) double sm[];
  const MlpP fm = p.fm[t], fv = p.fv[t], fe = p.fe[t];
  const bool nxt = t + 1 < p.L;
  double* Fm2 = sm;
  double* Fv1 = Fm2 + F;
  double* Fv2 = Fv1 + F;
  double* Fea = Fv2 + F;
  double* Feb = Fea + F;
  double* Fna = Feb + F;
  double* Fnb = Fna + F;
  double* b1 = Fnb + F;
  double* cc = b1 + DP;
  double* b2 = cc + DP;
  double* vb1 = b2 + DP;
  double* vb2 = vb1 + DP;
  stage_frag<D>(Fm2, fm.W2, 0);
  stage_frag<D>(Fv1, fv.W1, 0);
  stage_frag<D>(Fv2, fv.W2, 0);
  stage_frag<D>(Fea, fe.W1, 0);
  stage_frag<D>(Feb, fe.W1, D);
  if (nxt) {
    stage_frag<D>(Fna, p.fm[t + 1].W1, 0);
    stage_frag<D>(Fnb, p.fm[t + 1].W1, D);
  }
  stage_vec<D>(b1, fm.b1);
  stage_vec<D>(cc, fm.W1 + 2 * D * D);  // edge-feature row of W1m (d_edge == 1)
  stage_vec<D>(b2, fm.b2);
  stage_vec<D>(vb1, fv.b1);
  stage_vec<D>(vb2, fv.b2);
  __syncthreads();
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t base = (int64_t)(blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 8; base < n; base += warps * 8) {
    const int64_t i = base + r;
    const bool ok = i < n;
    const int64_t ic = ok ? i : n - 1;
    double S_[KS], pi[KS], cv[KS];
    load_row(pi, PQ + ic * 2 * DP, c, KS);
#pragma unroll
    for (int v = 0; v < KS; ++v) {
      const int f = feat(v, c);
      S_[v] = 0.0;
      pi[v] += b1[f];
      cv[v] = cc[f];
    }
    const int32_t lo = offs[ic], hi = ok ? offs[ic + 1] : lo;
    // neighbours in batches of NBAT: all their index / edge-feature loads, then all their Q rows,
    // are in flight together (same summation order as one at a time)
#ifndef SG_NODE_NBAT
#define SG_NODE_NBAT 5
#endif
    constexpr int NBAT = SG_NODE_NBAT;
    for (int32_t k0 = lo; k0 < hi; k0 += NBAT) {
      int64_t jn[NBAT];
      double e[NBAT];
#pragma unroll
      for (int u = 0; u < NBAT; ++u) {
        const int32_t kk = k0 + u < hi ? k0 + u : k0;
        jn[u] = cols[kk];
        e[u] = ef[kk];
      }
      double q[NBAT][KS];
#pragma unroll
      for (int u = 0; u < NBAT; ++u) load_row(q[u], PQ + jn[u] * 2 * DP + DP, c, KS);
#pragma unroll
      for (int u = 0; u < NBAT; ++u)
        if (k0 + u < hi) {
#pragma unroll
          for (int v = 0; v < KS; ++v) S_[v] += act_fn<ACT>(pi[v] + q[u][v] + e[u] * cv[v]);
        }
    }
    const double deg = (double)(hi - lo);
    double m[KS], u[KS];
#pragma unroll
    for (int v = 0; v < KS; ++v) { const int f = feat(v, c); m[v] = deg * b2[f]; u[v] = vb1[f]; }
    mv<D>(S_, Fm2, m, lane);
    mv<D>(m, Fv1, u, lane);
    double xo[KS];
    load_row(xo, X + ic * DP, c, KS);
#pragma unroll
    for (int v = 0; v < KS; ++v) { u[v] = act_fn<ACT>(u[v]); xo[v] += vb2[feat(v, c)]; }
    mv<D>(u, Fv2, xo, lane);  // xo = X + f_v(m): the updated node state
    if (ok) {
#pragma unroll
      for (int nb = 0; nb < KS / 2; ++nb)
        *reinterpret_cast<double2*>(X + i * DP + 8 * nb + 2 * c) = make_double2(xo[2 * nb], xo[2 * nb + 1]);
    }
    double* ep = EPQ + ((int64_t)t * n) * 2 * DP;
    const double* Fs[4] = {Fea, Feb, Fna, Fnb};
    double* dstb[4] = {ep, ep + DP, PQn, PQn + DP};
    const int nout = nxt ? 4 : 2;
    for (int o = 0; o < nout; ++o) {
#pragma unroll
      for (int v = 0; v < KS; ++v) u[v] = 0.0;
      mv<D>(xo, Fs[o], u, lane);
      if (ok) {
#pragma unroll
        for (int nb = 0; nb < KS / 2; ++nb)
          *reinterpret_cast<double2*>(dstb[o] + i * 2 * DP + 8 * nb + 2 * c) = make_double2(u[2 * nb], u[2 * nb + 1]);
      }
    }
  }
}

// ------------------------------------------------------------------ fused edge pass
// Shared memory: per layer [We1c frag][We2 frag][be1][be2]; then [Ee2 frag][D1 frag]
// [Ee1][eb1][eb2][bd1][D2] (padded vectors) and the scalar bd2.
template <int D>
__host__ __device__ constexpr int edge_smem_doubles(int L) {
  return L * (2 * Shape<D>::FRAG + 2 * Shape<D>::DP) + 2 * Shape<D>::FRAG + 5 * Shape<D>::DP + 2;
}

template <int D, int ACT>
__global__ void __launch_bounds__(256) k_edge_pass(GnnP p, int64_t nnz, const int32_t* __restrict__ rows,
                                                   const int32_t* __restrict__ cols,
                                                   const double* __restrict__ ef,
                                                   const double* __restrict__ EPQ, int64_t n,
                                                   double* __restrict__ g) {
  using S = Shape<D>;
  constexpr int DP = S::DP, KS = S::KS, F = S::FRAG;
  extern __shared__ __align__(16) double w[];
  const int L = p.L;
  const int per = 2 * F + 2 * DP;
  for (int t = 0; t < L; ++t) {
    double* base = w + t * per;
    stage_frag<D>(base, p.fe[t].W1, 2 * D);
    stage_frag<D>(base + F, p.fe[t].W2, 0);
    stage_vec<D>(base + 2 * F, p.fe[t].b1);
    stage_vec<D>(base + 2 * F + DP, p.fe[t].b2);
  }
  double* FE2 = w + L * per;
  double* FD1 = FE2 + F;
  double* e1 = FD1 + F;
  double* eb1 = e1 + DP;
  double* eb2 = eb1 + DP;
  double* db1 = eb2 + DP;
  double* d2 = db1 + DP;
  double* db2 = d2 + DP;
  stage_frag<D>(FE2, p.ee.W2, 0);
  stage_frag<D>(FD1, p.dec.W1, 0);
  stage_vec<D>(e1, p.ee.W1);
  stage_vec<D>(eb1, p.ee.b1);
  stage_vec<D>(eb2, p.ee.b2);
  stage_vec<D>(db1, p.dec.b1);
  stage_vec<D>(d2, p.dec.W2);
  if (threadIdx.x == 0) db2[0] = p.dec.b2[0];
  __syncthreads();
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t base = (int64_t)(blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 8; base < nnz; base += warps * 8) {
    const int64_t k = base + r;
    const bool ok = k < nnz;
    const int64_t kc = ok ? k : nnz - 1;
    const double e = ef[kc];
    const int64_t i = rows[kc], j = cols[kc];
    double h[KS], a[KS];
#pragma unroll
    for (int v = 0; v < KS; ++v) {
      const int f = feat(v, c);
      a[v] = act_fn<ACT>(fma(e, e1[f], eb1[f]));
      h[v] = eb2[f];
    }
    // layer t's P_i / Q_j rows are loaded during layer t-1's products (3 CTAs/SM at 78
    // registers beat 4 CTAs/SM loading them on demand: C2 factor build 31.0 -> 30.1 ms)
    double pn[KS], qn[KS];
    if (L > 0) {
      load_row(pn, EPQ + i * 2 * DP, c, KS);
      load_row(qn, EPQ + j * 2 * DP + DP, c, KS);
    }
    mv<D>(a, FE2, h, lane);
    for (int t = 0; t < L; ++t) {
      const double* lay = w + t * per;
      double q[KS];
#pragma unroll
      for (int v = 0; v < KS; ++v) { a[v] = pn[v]; q[v] = qn[v]; }
      if (t + 1 < L) {
        const double* Pn = EPQ + (int64_t)(t + 1) * n * 2 * DP;
        load_row(pn, Pn + i * 2 * DP, c, KS);
        load_row(qn, Pn + j * 2 * DP + DP, c, KS);
      }
#pragma unroll
      for (int v = 0; v < KS; ++v) a[v] += q[v] + lay[2 * F + feat(v, c)];
      mv<D>(h, lay, a, lane);
#pragma unroll
      for (int v = 0; v < KS; ++v) { a[v] = act_fn<ACT>(a[v]); h[v] += lay[2 * F + DP + feat(v, c)]; }
      mv<D>(a, lay + F, h, lane);
    }
#pragma unroll
    for (int v = 0; v < KS; ++v) a[v] = db1[feat(v, c)];
    mv<D>(h, FD1, a, lane);
    double part = 0.0;
#pragma unroll
    for (int v = 0; v < KS; ++v) part = fma(act_fn<ACT>(a[v]), d2[feat(v, c)], part);
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    if (ok && c == 0) g[k] = part + db2[0];
  }
}

// ------------------------------------------------------------------ edge pass on tcgen05
// The same per-edge computation in fp32 on the 5th-generation tensor core: a CTA of 128 threads
// owns a tile of 128 edges (thread = edge = accumulator row / TMEM lane), and every [128 x D] .
// [D x D] product of the edge MLPs is kind::tf32 tcgen05.mma with the 3xTF32 split (a_hi b_hi +
// a_hi b_lo + a_lo b_hi, fp32 accumulate in TMEM): the activations are written K-major into
// shared memory by their threads, one elected thread issues the MMAs, tcgen05.commit arrives on
// an mbarrier, and every thread reads its row back with tcgen05.ld.  Weights (hi / lo splits) stay
// in shared memory for the CTA's life; the fp64 node path's P'_t / Q'_t rows are read and rounded
// to fp32 per edge.  Accuracy: ~fp32 (north_star: G within 1e-5 in fp32) -- the fp64 DMMA edge
// pass stays the default; this one is opt-in (`edge_mode` 1).
template <int D>
struct TcEdge {
  static constexpr int KP = (D + 7) / 8 * 8;       // padded K (multiple of the MMA's 8)
  static constexpr int NP = 32;                     // padded N (TMEM columns)
  static constexpr int BW = NP * KP;                // floats per weight matrix (one split)
  static constexpr int AW = 128 * KP;               // floats per activation tile (one split)
  static constexpr int NV = 24;                     // padded vector length (<= 32)
  __host__ __device__ static int nmat(int L) { return 2 + 2 * L; }  // FE2, D1, per layer We1c, We2
  static size_t smem(int L) {
    return (size_t)(2 * nmat(L) * BW + 2 * AW) * sizeof(float) + (size_t)(5 + 2 * L) * 32 * sizeof(float) + 64;
  }
};

template <int D, int ACT>
__global__ void __launch_bounds__(128, 2) k_edge_pass_tc(GnnP p, int64_t nnz, const int32_t* __restrict__ rows,
                                                         const int32_t* __restrict__ cols,
                                                         const double* __restrict__ ef,
                                                         const double* __restrict__ EPQ, int64_t n,
                                                         double* __restrict__ g) {
  using T = TcEdge<D>;
  constexpr int KP = T::KP, BW = T::BW, AW = T::AW, DP = Shape<D>::DP;
  static_assert(KP <= 32 && D <= 32, "tensor-core edge pass: hidden size <= 32");
  extern __shared__ __align__(128) float smf[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int L = p.L;
  const int tid = threadIdx.x, warp = tid >> 5;
  float* Bw = smf;                               // [nmat][2][BW] weight splits, B operand layout
  float* Ah = Bw + 2 * T::nmat(L) * BW;          // [AW] activation tile, hi split
  float* Al = Ah + AW;                           // [AW] lo split
  float* vec = Al + AW;                          // [5 + 2L][32]: e1, eb1, eb2, db1, d2, be1_t, be2_t
  // matrix m: 0 = FE2 (ee.W2), 1 = D1 (dec.W1), 2 + 2t = We1c_t (fe[t].W1 rows 2D..3D), 3 + 2t = We2_t
  auto wsrc = [&](int m) -> const double* {
    if (m == 0) return p.ee.W2;
    if (m == 1) return p.dec.W1;
    const int t = (m - 2) >> 1;
    return ((m - 2) & 1) ? p.fe[t].W2 : p.fe[t].W1 + 2 * D * D;
  };
  for (int m = 0; m < T::nmat(L); ++m) {
    const double* W = wsrc(m);
    for (int idx = tid; idx < T::NP * KP; idx += 128) {
      const int nn = idx / KP, k = idx % KP;
      const float w = (nn < D && k < D) ? (float)W[k * D + nn] : 0.f;
      const float hi = tf32_rn(w), lo = tf32_rn(w - hi);
      Bw[(2 * m) * BW + umma_off(nn, k, T::NP) / 4] = hi;
      Bw[(2 * m + 1) * BW + umma_off(nn, k, T::NP) / 4] = lo;
    }
  }
  for (int f = tid; f < 32; f += 128) {
    const bool in = f < D;
    vec[0 * 32 + f] = in ? (float)p.ee.W1[f] : 0.f;
    vec[1 * 32 + f] = in ? (float)p.ee.b1[f] : 0.f;
    vec[2 * 32 + f] = in ? (float)p.ee.b2[f] : 0.f;
    vec[3 * 32 + f] = in ? (float)p.dec.b1[f] : 0.f;
    vec[4 * 32 + f] = in ? (float)p.dec.W2[f] : 0.f;
    for (int t = 0; t < L; ++t) {
      vec[(5 + 2 * t) * 32 + f] = in ? (float)p.fe[t].b1[f] : 0.f;
      vec[(6 + 2 * t) * 32 + f] = in ? (float)p.fe[t].b2[f] : 0.f;
    }
  }
  const float db2 = (float)p.dec.b2[0];
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&tmem_base, T::NP);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tmem_base;
  const uint32_t my_lanes = taddr + ((uint32_t)(warp * 32) << 16);
  constexpr uint32_t idesc = umma_idesc_tf32(128, T::NP);
  uint32_t phase = 0;
  // out = act_in[128 x D] . W_m  (3xTF32), every thread its own row
  auto gemm = [&](const float (&x)[32], int m, float (&out)[32]) {
#pragma unroll
    for (int c = 0; c < KP / 4; ++c) {
      float4 hi, lo;
      float* hp = &hi.x;
      float* lp = &lo.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float v = x[4 * c + e];
        hp[e] = tf32_rn(v);
        lp[e] = tf32_rn(v - hp[e]);
      }
      const uint32_t o = umma_off(tid, 4 * c, 128) / 4;
      *reinterpret_cast<float4*>(Ah + o) = hi;
      *reinterpret_cast<float4*>(Al + o) = lo;
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();  // the tile is complete; every thread's previous TMEM read has finished
    tc_fence_after();
    if (tid == 0) {
      const float* bh = Bw + (2 * m) * BW;
      const float* bl = Bw + (2 * m + 1) * BW;
#pragma unroll
      for (int s = 0; s < KP / 8; ++s) {
        const uint64_t dah = umma_desc(smem_u32(Ah) + s * 2 * 128 * 16, 128 * 16, 128);
        const uint64_t dal = umma_desc(smem_u32(Al) + s * 2 * 128 * 16, 128 * 16, 128);
        const uint64_t dbh = umma_desc(smem_u32(bh) + s * 2 * T::NP * 16, T::NP * 16, 128);
        const uint64_t dbl = umma_desc(smem_u32(bl) + s * 2 * T::NP * 16, T::NP * 16, 128);
        umma_tf32(taddr, dah, dbh, idesc, s > 0);
        umma_tf32(taddr, dah, dbl, idesc, true);
        umma_tf32(taddr, dal, dbh, idesc, true);
      }
      umma_commit(&bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1u;
    tc_fence_after();
    tmem_ld32(my_lanes, out);
  };
  for (int64_t tile = blockIdx.x; tile * 128 < nnz; tile += gridDim.x) {
    const int64_t k = tile * 128 + tid;
    const bool ok = k < nnz;
    const int64_t kc = ok ? k : nnz - 1;
    const float e = (float)ef[kc];
    const int64_t i = rows[kc], j = cols[kc];
    float a[32], h[32], v[32];
#pragma unroll
    for (int f = 0; f < 32; ++f) a[f] = f < D ? act_fn<ACT>(fmaf(e, vec[f], vec[32 + f])) : 0.f;
    gemm(a, 0, v);
#pragma unroll
    for (int f = 0; f < 32; ++f) h[f] = f < D ? v[f] + vec[64 + f] : 0.f;
    for (int t = 0; t < L; ++t) {
      const double* Pt = EPQ + ((int64_t)t * n) * 2 * DP;
      const double* pr = Pt + i * 2 * DP;
      const double* qr = Pt + j * 2 * DP + DP;
      gemm(h, 2 + 2 * t, v);
      const float* b1 = vec + (5 + 2 * t) * 32;
      const float* b2 = vec + (6 + 2 * t) * 32;
#pragma unroll
      for (int f = 0; f < 32; f += 2) {
        if (f < D) {
          const double2 pp = *reinterpret_cast<const double2*>(pr + f);
          const double2 qq = *reinterpret_cast<const double2*>(qr + f);
          a[f] = act_fn<ACT>((float)(pp.x + qq.x) + b1[f] + v[f]);
          a[f + 1] = f + 1 < D ? act_fn<ACT>((float)(pp.y + qq.y) + b1[f + 1] + v[f + 1]) : 0.f;
        } else {
          a[f] = a[f + 1] = 0.f;
        }
      }
      gemm(a, 3 + 2 * t, v);
#pragma unroll
      for (int f = 0; f < 32; ++f) h[f] = f < D ? h[f] + (v[f] + b2[f]) : 0.f;
    }
    gemm(h, 1, v);
    float part = 0.f;
#pragma unroll
    for (int f = 0; f < 32; ++f)
      if (f < D) part = fmaf(act_fn<ACT>(v[f] + vec[96 + f]), vec[128 + f], part);
    if (ok) g[k] = (double)(part + db2);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(taddr, T::NP);
}

template <class K>
static int resident(K kernel, int threads, size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  return per_sm;
}

static int grid_for(int64_t rows, int per_sm, int warps = 4) {
  const int64_t groups = (rows + 7) / 8;       // 8 rows per warp
  int64_t b = (groups + warps - 1) / warps;    // warps per CTA
  const int64_t cap = 148LL * per_sm;
  return (int)(b > cap ? cap : (b < 1 ? 1 : b));
}

template <int D, int ACT>
int run_forward(const GnnP& p, int64_t n, int64_t nnz, const int32_t* offs, const int32_t* cols,
                const int32_t* rows, const double* V, const double* ef, double* g, double* X,
                double* PQa, double* PQb, double* EPQ, cudaStream_t s, int edge_mode = 0) {
  using S = Shape<D>;
  const size_t sm_enc = (size_t)(6 * S::DP + 3 * S::FRAG + 16) * sizeof(double);
  SG_CUDA(cudaFuncSetAttribute(k_node_encode<D, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_enc));
  k_node_encode<D, ACT><<<grid_for(n, resident(k_node_encode<D, ACT>, 128, sm_enc)), 128, sm_enc, s>>>(p, n, V, X, PQa);
  SG_LAUNCH_CHECK("k_node_encode");
  const size_t sm_layer = (size_t)(node_layer_smem_doubles<D>() + 16) * sizeof(double);
  SG_CUDA(cudaFuncSetAttribute(k_node_layer<D, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_layer));
  const int layer_res = resident(k_node_layer<D, ACT>, 128, sm_layer);
  double* cur = PQa;
  double* nxt = PQb;
  for (int t = 0; t < p.L; ++t) {
    k_node_layer<D, ACT><<<grid_for(n, layer_res), 128, sm_layer, s>>>(p, t, n, offs, cols, ef, X, cur, nxt, EPQ);
    SG_LAUNCH_CHECK("k_node_layer");
    double* tmp = cur; cur = nxt; nxt = tmp;
  }
  if (edge_mode == 1) {  // tcgen05 3xTF32 edge pass
    if constexpr (TcEdge<D>::KP <= 32) {
      const size_t smt = TcEdge<D>::smem(p.L);
      if (smt > 227 * 1024) {
        set_error("tensor-core edge pass: weights (%zu bytes) exceed shared memory", smt);
        return SG_EUNSUPPORTED;
      }
      SG_CUDA(cudaFuncSetAttribute(k_edge_pass_tc<D, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smt));
      const int64_t tiles = (nnz + 127) / 128;
      const int res = resident(k_edge_pass_tc<D, ACT>, 128, smt);
      const int64_t cap = 148LL * res;
      k_edge_pass_tc<D, ACT><<<(unsigned)(tiles < cap ? tiles : cap), 128, smt, s>>>(p, nnz, rows, cols, ef, EPQ, n, g);
      SG_LAUNCH_CHECK("k_edge_pass_tc");
      return SG_OK;
    }
  }
  const size_t smem = (edge_smem_doubles<D>(p.L) + 16) * sizeof(double);
  if (smem > 227 * 1024) {
    set_error("edge-pass weights (%zu bytes) exceed shared memory; reduce n_layers or hidden_dim", smem);
    return SG_EUNSUPPORTED;
  }
  SG_CUDA(cudaFuncSetAttribute(k_edge_pass<D, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // 8 warps per CTA share one copy of the edge weights in shared memory; the grid-stride grid is
  // exactly the co-resident CTAs (a partial second wave would double the tail)
  k_edge_pass<D, ACT><<<grid_for(nnz, resident(k_edge_pass<D, ACT>, 256, smem), 8), 256, smem, s>>>(
      p, nnz, rows, cols, ef, EPQ, n, g);
  SG_LAUNCH_CHECK("k_edge_pass");
  return SG_OK;
}

template <int ACT>
int dispatch_hidden(int hidden, const GnnP& p, int64_t n, int64_t nnz, const int32_t* offs,
                    const int32_t* cols, const int32_t* rows, const double* V, const double* ef,
                    double* g, double* X, double* PQa, double* PQb, double* EPQ, cudaStream_t s,
                    int edge_mode) {
#define SG_H(DD) \
  case DD: return run_forward<DD, ACT>(p, n, nnz, offs, cols, rows, V, ef, g, X, PQa, PQb, EPQ, s, edge_mode);
  switch (hidden) {
    SG_H(4) SG_H(6) SG_H(8) SG_H(12) SG_H(16) SG_H(24) SG_H(32)
  }
#undef SG_H
  set_error("hidden_dim %d not compiled (supported: 4,6,8,12,16,24,32)", hidden);
  return SG_EUNSUPPORTED;
}

}  // namespace sg

using namespace sg;

extern "C" int sg_gnn_forward_ex(const double* params, int64_t n_params, int n_layers, int hidden,
                                 int d_node, int d_edge, int act, int64_t n, int64_t nnz,
                                 const int32_t* offs, const int32_t* cols, const int32_t* rows,
                                 const double* node_feat, const double* edge_feat, double* g_out,
                                 int32_t edge_mode, void* ws, size_t* ws_bytes, void* stream) {
  const int64_t D = hidden, L = n_layers, DP = (hidden + 7) / 8 * 8;
  Carve c(ws);
  double* X = c.take<double>(n * DP);
  double* PQa = c.take<double>(n * 2 * DP);
  double* PQb = c.take<double>(n * 2 * DP);
  double* EPQ = c.take<double>((L > 0 ? L : 1) * n * 2 * DP);
  if (!ws) { *ws_bytes = c.off; return SG_OK; }
  if (*ws_bytes < c.off) { set_error("workspace too small"); return SG_EINVAL; }
  if (d_edge != 1) { set_error("d_edge must be 1 on the GPU path"); return SG_EUNSUPPORTED; }
  if (d_node < 1 || d_node > 4) { set_error("d_node must be in [1, 4] on the GPU path"); return SG_EUNSUPPORTED; }
  if (n_layers < 0 || n_layers > 16) { set_error("n_layers must be in [0, 16] on the GPU path"); return SG_EUNSUPPORTED; }
  if (act != 0 && act != 1) { set_error("activation must be relu (0) or tanh (1)"); return SG_EINVAL; }
  // parameter layout (gnn.py:130-136 declaration order, mlp_hidden_layers == 1)
  auto mlp_size = [&](int64_t din, int64_t dout) { return din * D + D + D * dout + dout; };
  const int64_t want = mlp_size(d_node, D) + mlp_size(d_edge, D) +
                       L * (mlp_size(2 * D + d_edge, D) + mlp_size(D, D) + mlp_size(3 * D, D)) +
                       mlp_size(D, 1);
  if (want != n_params) {
    set_error("parameter count %lld does not match a 1-hidden-layer model (%lld)",
              (long long)n_params, (long long)want);
    return SG_EUNSUPPORTED;
  }
  GnnP p{};
  p.L = n_layers;
  p.dn = d_node;
  const double* q = params;
  auto take_mlp = [&](int64_t din, int64_t dout) {
    MlpP m;
    m.W1 = q; q += din * D;
    m.b1 = q; q += D;
    m.W2 = q; q += D * dout;
    m.b2 = q; q += dout;
    return m;
  };
  p.en = take_mlp(d_node, D);
  p.ee = take_mlp(d_edge, D);
  for (int t = 0; t < n_layers; ++t) {
    p.fm[t] = take_mlp(2 * D + d_edge, D);
    p.fv[t] = take_mlp(D, D);
    p.fe[t] = take_mlp(3 * D, D);
  }
  p.dec = take_mlp(D, 1);
  if (n == 0 || nnz == 0) return SG_OK;
  cudaStream_t s = as_stream(stream);
  if (edge_mode < 0 || edge_mode > 1) { set_error("edge_mode must be 0 (fp64 DMMA) or 1 (tcgen05 3xTF32)"); return SG_EINVAL; }
  if (act == 0)
    return dispatch_hidden<0>(hidden, p, n, nnz, offs, cols, rows, node_feat, edge_feat, g_out, X, PQa, PQb, EPQ, s,
                              edge_mode);
  return dispatch_hidden<1>(hidden, p, n, nnz, offs, cols, rows, node_feat, edge_feat, g_out, X, PQa, PQb, EPQ, s,
                            edge_mode);
}

extern "C" int sg_gnn_forward(const double* params, int64_t n_params, int n_layers, int hidden,
                              int d_node, int d_edge, int act, int64_t n, int64_t nnz,
                              const int32_t* offs, const int32_t* cols, const int32_t* rows,
                              const double* node_feat, const double* edge_feat, double* g_out,
                              void* ws, size_t* ws_bytes, void* stream) {
  return sg_gnn_forward_ex(params, n_params, n_layers, hidden, d_node, d_edge, act, n, nnz, offs, cols, rows,
                           node_feat, edge_feat, g_out, 0, ws, ws_bytes, stream);
}
