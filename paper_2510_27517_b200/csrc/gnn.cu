// GNN forward (gnn.py:208-253) restructured for the GPU.
//
// With message_uses_hidden_edge = False the node path never reads the edge state H, and the
// first layer of every MLP on a concatenation is linear.  So
//   * node path, per layer t: P = X W1m[0:D], Q = X W1m[D:2D] are node-level products; the
//     message MLP's hidden activations are summed per CSR row, act(P_i + Q_j + e_k c + b1),
//     and its (linear) second layer is applied AFTER the row sum: m = S W2m + deg b2m;
//     X += f_v(m).  One kernel per layer, thread per row, fused with the node-level products
//     the next stages need (P'_t, Q'_t for the edge pass; P, Q for layer t+1).
//   * edge pass: ONE kernel, thread per edge, h kept in registers through all L layers:
//     h = E_e(e); h += f_e-second-layer(act(P'_t[i] + Q'_t[j] + h W1e[2D:3D] + b1e)); g = D(h).
//     H never touches HBM (the reference tape holds ~18 KB per edge).
// Node-level arrays are structure-of-arrays ([feature][node]) so the per-edge gathers of a
// warp (consecutive edges of a few consecutive rows) coalesce.  All MLP weights a kernel needs
// are staged once per CTA in shared memory and read as 16-byte broadcasts.
// All arithmetic is fp64 (FMA allowed; parity is tolerance-based: OpenBLAS DGEMM order differs).
#include "common.cuh"

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

// out[j] (+)= sum_k in[k] * W[k*DO + j] with W in shared memory (16-byte loads, DO even).
template <int DI, int DO, bool ACC>
__device__ __forceinline__ void mv(const double* in, const double* __restrict__ W, double* out) {
  if (!ACC) {
#pragma unroll
    for (int j = 0; j < DO; ++j) out[j] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < DI; ++k) {
    const double v = in[k];
    const double2* w2 = reinterpret_cast<const double2*>(W + k * DO);
#pragma unroll
    for (int j = 0; j < DO / 2; ++j) {
      const double2 w = w2[j];
      out[2 * j] = fma(v, w.x, out[2 * j]);
      out[2 * j + 1] = fma(v, w.y, out[2 * j + 1]);
    }
  }
}

// Cooperative global -> shared copy (doubles), returns the next free offset.
__device__ __forceinline__ int stage(double* sm, int off, const double* src, int cnt) {
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) sm[off + k] = src[k];
  return off + ((cnt + 1) & ~1);  // keep 16-byte alignment for the next block
}

// ------------------------------------------------------------------ node encoder
// X = E_n(V); PQ = [X W1m0[0:D] ; X W1m0[D:2D]] (layer 0's node products).  SoA outputs.
template <int D, int ACT>
__global__ void __launch_bounds__(128) k_node_encode(GnnP p, int64_t n, const double* __restrict__ V,
                                                     double* __restrict__ X, double* __restrict__ PQ) {
  extern __shared__ __align__(16) double sm[];
  int o = 0;
  const int oW1 = o; o = stage(sm, o, p.en.W1, p.dn * D);
  const int ob1 = o; o = stage(sm, o, p.en.b1, D);
  const int oW2 = o; o = stage(sm, o, p.en.W2, D * D);
  const int ob2 = o; o = stage(sm, o, p.en.b2, D);
  const int oP = o; if (p.L > 0) o = stage(sm, o, p.fm[0].W1, 2 * D * D);
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double h[D], x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) h[j] = sm[ob1 + j];
    for (int k = 0; k < p.dn; ++k) {
      const double v = V[i * p.dn + k];
#pragma unroll
      for (int j = 0; j < D; ++j) h[j] = fma(v, sm[oW1 + k * D + j], h[j]);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) { h[j] = act_fn<ACT>(h[j]); x[j] = sm[ob2 + j]; }
    mv<D, D, true>(h, sm + oW2, x);
#pragma unroll
    for (int j = 0; j < D; ++j) X[(int64_t)j * n + i] = x[j];
    if (p.L > 0) {
      double q[D];
      mv<D, D, false>(x, sm + oP, q);
#pragma unroll
      for (int j = 0; j < D; ++j) PQ[(int64_t)j * n + i] = q[j];
      mv<D, D, false>(x, sm + oP + D * D, q);
#pragma unroll
      for (int j = 0; j < D; ++j) PQ[(int64_t)(D + j) * n + i] = q[j];
    }
  }
}

// ------------------------------------------------------------------ node layer t
template <int D>
__host__ __device__ constexpr int node_layer_smem_doubles() {
  return 7 * D * D + 8 * D;
}

template <int D, int ACT>
__global__ void __launch_bounds__(128) k_node_layer(GnnP p, int t, int64_t n, const int32_t* __restrict__ offs,
                                                    const int32_t* __restrict__ cols,
                                                    const double* __restrict__ ef, double* __restrict__ X,
                                                    const double* __restrict__ PQ, double* __restrict__ PQn,
                                                    double* __restrict__ EPQ) {
  extern __shared__ __align__(16) double sm[];
  const MlpP fm = p.fm[t], fv = p.fv[t], fe = p.fe[t];
  const bool nxt = t + 1 < p.L;
  int o = 0;
  const int o_b1 = o; o = stage(sm, o, fm.b1, D);
  const int o_c = o; o = stage(sm, o, fm.W1 + 2 * D * D, D);  // edge-feature row (d_edge == 1)
  const int o_W2 = o; o = stage(sm, o, fm.W2, D * D);
  const int o_b2 = o; o = stage(sm, o, fm.b2, D);
  const int o_V1 = o; o = stage(sm, o, fv.W1, D * D);
  const int o_vb1 = o; o = stage(sm, o, fv.b1, D);
  const int o_V2 = o; o = stage(sm, o, fv.W2, D * D);
  const int o_vb2 = o; o = stage(sm, o, fv.b2, D);
  const int o_E = o; o = stage(sm, o, fe.W1, 2 * D * D);
  const int o_N = o; if (nxt) o = stage(sm, o, p.fm[t + 1].W1, 2 * D * D);
  __syncthreads();
  const double* P = PQ;
  const double* Q = PQ + (int64_t)D * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double S[D], pi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { S[j] = 0.0; pi[j] = P[(int64_t)j * n + i] + sm[o_b1 + j]; }
    const int32_t lo = offs[i], hi = offs[i + 1];
    for (int32_t k = lo; k < hi; ++k) {
      const int64_t jn = cols[k];
      const double e = ef[k];
#pragma unroll
      for (int j = 0; j < D; ++j) S[j] += act_fn<ACT>(pi[j] + Q[(int64_t)j * n + jn] + e * sm[o_c + j]);
    }
    const double deg = (double)(hi - lo);
    double m[D];
#pragma unroll
    for (int j = 0; j < D; ++j) m[j] = deg * sm[o_b2 + j];
    mv<D, D, true>(S, sm + o_W2, m);
    double u[D];
#pragma unroll
    for (int j = 0; j < D; ++j) u[j] = sm[o_vb1 + j];
    mv<D, D, true>(m, sm + o_V1, u);
#pragma unroll
    for (int j = 0; j < D; ++j) { u[j] = act_fn<ACT>(u[j]); m[j] = X[(int64_t)j * n + i] + sm[o_vb2 + j]; }
    mv<D, D, true>(u, sm + o_V2, m);  // m now holds the updated X row
#pragma unroll
    for (int j = 0; j < D; ++j) X[(int64_t)j * n + i] = m[j];
    double* ep = EPQ + (int64_t)t * 2 * D * n;
    mv<D, D, false>(m, sm + o_E, u);
#pragma unroll
    for (int j = 0; j < D; ++j) ep[(int64_t)j * n + i] = u[j];
    mv<D, D, false>(m, sm + o_E + D * D, u);
#pragma unroll
    for (int j = 0; j < D; ++j) ep[(int64_t)(D + j) * n + i] = u[j];
    if (nxt) {
      mv<D, D, false>(m, sm + o_N, u);
#pragma unroll
      for (int j = 0; j < D; ++j) PQn[(int64_t)j * n + i] = u[j];
      mv<D, D, false>(m, sm + o_N + D * D, u);
#pragma unroll
      for (int j = 0; j < D; ++j) PQn[(int64_t)(D + j) * n + i] = u[j];
    }
  }
}

// ------------------------------------------------------------------ fused edge pass
// Edge-path weights in shared memory:
//   [Ee1 D][be1 D][Ee2 DxD][be2 D] + L x ([We1c DxD][be1 D][We2 DxD][be2 D]) + [D1 DxD][bd1 D][D2 D][bd2 1]
template <int D>
__host__ __device__ constexpr int edge_smem_doubles(int L) {
  return (3 * D + D * D) + L * (2 * D * D + 2 * D) + (D * D + 2 * D + 2);
}

template <int D, int ACT>
__global__ void __launch_bounds__(128) k_edge_pass(GnnP p, int64_t nnz, const int32_t* __restrict__ rows,
                                                   const int32_t* __restrict__ cols,
                                                   const double* __restrict__ ef,
                                                   const double* __restrict__ EPQ, int64_t n,
                                                   double* __restrict__ g) {
  extern __shared__ __align__(16) double w[];
  const int L = p.L;
  int o = 0;
  o = stage(w, o, p.ee.W1, D); o = stage(w, o, p.ee.b1, D); o = stage(w, o, p.ee.W2, D * D);
  o = stage(w, o, p.ee.b2, D);
  for (int t = 0; t < L; ++t) {
    o = stage(w, o, p.fe[t].W1 + 2 * D * D, D * D); o = stage(w, o, p.fe[t].b1, D);
    o = stage(w, o, p.fe[t].W2, D * D); o = stage(w, o, p.fe[t].b2, D);
  }
  const int o_dec = o;
  o = stage(w, o, p.dec.W1, D * D); o = stage(w, o, p.dec.b1, D); o = stage(w, o, p.dec.W2, D);
  o = stage(w, o, p.dec.b2, 1);
  __syncthreads();
  const double* Ee1 = w;
  const double* eb1 = w + D;
  const double* Ee2 = w + 2 * D;
  const double* eb2 = w + 2 * D + D * D;
  const double* lay = w + 3 * D + D * D;
  const double* dec = w + o_dec;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const double e = ef[k];
    const int64_t i = rows[k], j = cols[k];
    double h[D], a[D];
#pragma unroll
    for (int q = 0; q < D; ++q) { a[q] = act_fn<ACT>(fma(e, Ee1[q], eb1[q])); h[q] = eb2[q]; }
    mv<D, D, true>(a, Ee2, h);
    for (int t = 0; t < L; ++t) {
      const double* W1c = lay + t * (2 * D * D + 2 * D);
      const double* b1 = W1c + D * D;
      const double* W2 = b1 + D;
      const double* b2 = W2 + D * D;
      const double* Pt = EPQ + (int64_t)t * 2 * D * n;
#pragma unroll
      for (int q = 0; q < D; ++q) a[q] = Pt[(int64_t)q * n + i] + Pt[(int64_t)(D + q) * n + j] + b1[q];
      mv<D, D, true>(h, W1c, a);
#pragma unroll
      for (int q = 0; q < D; ++q) { a[q] = act_fn<ACT>(a[q]); h[q] += b2[q]; }
      mv<D, D, true>(a, W2, h);
    }
#pragma unroll
    for (int q = 0; q < D; ++q) a[q] = dec[D * D + q];
    mv<D, D, true>(h, dec, a);
    double out = dec[D * D + 2 * D];
#pragma unroll
    for (int q = 0; q < D; ++q) out = fma(act_fn<ACT>(a[q]), dec[D * D + D + q], out);
    g[k] = out;
  }
}

static int grid_for(int64_t n, int threads, int per_sm) {
  int64_t b = ceil_div(n > 0 ? n : 1, threads);
  const int64_t cap = 148LL * per_sm;
  return (int)(b > cap ? cap : b);
}

template <int D, int ACT>
int run_forward(const GnnP& p, int64_t n, int64_t nnz, const int32_t* offs, const int32_t* cols,
                const int32_t* rows, const double* V, const double* ef, double* g, double* X,
                double* PQa, double* PQb, double* EPQ, cudaStream_t s) {
  const size_t sm_enc = (size_t)(p.dn * D + 4 * D + D * D + 2 * D * D + 8) * sizeof(double);
  SG_CUDA(cudaFuncSetAttribute(k_node_encode<D, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_enc));
  k_node_encode<D, ACT><<<grid_for(n, 128, 16), 128, sm_enc, s>>>(p, n, V, X, PQa);
  SG_LAUNCH_CHECK("k_node_encode");
  const size_t sm_layer = (size_t)(node_layer_smem_doubles<D>() + 16) * sizeof(double);
  SG_CUDA(cudaFuncSetAttribute(k_node_layer<D, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_layer));
  double* cur = PQa;
  double* nxt = PQb;
  for (int t = 0; t < p.L; ++t) {
    k_node_layer<D, ACT><<<grid_for(n, 128, 16), 128, sm_layer, s>>>(p, t, n, offs, cols, ef, X, cur, nxt, EPQ);
    SG_LAUNCH_CHECK("k_node_layer");
    double* tmp = cur; cur = nxt; nxt = tmp;
  }
  const size_t smem = (edge_smem_doubles<D>(p.L) + 8 * (p.L + 4)) * sizeof(double);
  if (smem > 227 * 1024) {
    set_error("edge-pass weights (%zu bytes) exceed shared memory; reduce n_layers or hidden_dim", smem);
    return SG_EUNSUPPORTED;
  }
  SG_CUDA(cudaFuncSetAttribute(k_edge_pass<D, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_edge_pass<D, ACT><<<grid_for(nnz, 128, 16), 128, smem, s>>>(p, nnz, rows, cols, ef, EPQ, n, g);
  SG_LAUNCH_CHECK("k_edge_pass");
  return SG_OK;
}

template <int ACT>
int dispatch_hidden(int hidden, const GnnP& p, int64_t n, int64_t nnz, const int32_t* offs,
                    const int32_t* cols, const int32_t* rows, const double* V, const double* ef,
                    double* g, double* X, double* PQa, double* PQb, double* EPQ, cudaStream_t s) {
#define SG_H(DD) \
  case DD: return run_forward<DD, ACT>(p, n, nnz, offs, cols, rows, V, ef, g, X, PQa, PQb, EPQ, s);
  switch (hidden) {
    SG_H(4) SG_H(6) SG_H(8) SG_H(12) SG_H(16) SG_H(24) SG_H(32)
  }
#undef SG_H
  set_error("hidden_dim %d not compiled (supported: 4,6,8,12,16,24,32)", hidden);
  return SG_EUNSUPPORTED;
}

}  // namespace sg

using namespace sg;

extern "C" int sg_gnn_forward(const double* params, int64_t n_params, int n_layers, int hidden,
                              int d_node, int d_edge, int act, int64_t n, int64_t nnz,
                              const int32_t* offs, const int32_t* cols, const int32_t* rows,
                              const double* node_feat, const double* edge_feat, double* g_out,
                              void* ws, size_t* ws_bytes, void* stream) {
  const int64_t D = hidden, L = n_layers;
  Carve c(ws);
  double* X = c.take<double>(n * D);
  double* PQa = c.take<double>(n * 2 * D);
  double* PQb = c.take<double>(n * 2 * D);
  double* EPQ = c.take<double>((L > 0 ? L : 1) * n * 2 * D);
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
  if (act == 0)
    return dispatch_hidden<0>(hidden, p, n, nnz, offs, cols, rows, node_feat, edge_feat, g_out, X, PQa, PQb, EPQ, s);
  return dispatch_hidden<1>(hidden, p, n, nnz, offs, cols, rows, node_feat, edge_feat, g_out, X, PQa, PQb, EPQ, s);
}
