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
// All arithmetic is fp64 (FMA allowed; parity is tolerance-based: OpenBLAS DGEMM order differs).
// Weights live in shared memory; every thread of a warp reads the same weight element, so
// shared-memory reads are broadcasts.
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

// out[j] = b[j] + sum_k in[k] * W[k*ld + j], j < DO  (W in shared or global memory)
template <int DI, int DO>
__device__ __forceinline__ void matvec(const double* __restrict__ in, const double* __restrict__ W,
                                       const double* __restrict__ b, double* __restrict__ out, int ld) {
#pragma unroll
  for (int j = 0; j < DO; ++j) out[j] = b ? b[j] : 0.0;
#pragma unroll
  for (int k = 0; k < DI; ++k) {
    const double v = in[k];
#pragma unroll
    for (int j = 0; j < DO; ++j) out[j] = fma(v, W[k * ld + j], out[j]);
  }
}

// Node encoder, then P, Q of layer 1 (or nothing if L == 0).  X: [n x D], PQ: [n x 2D].
template <int D, int ACT>
__global__ void k_node_encode(GnnP p, int64_t n, const double* __restrict__ V, double* X, double* PQ) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double h[D], x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) h[j] = p.en.b1[j];
    for (int k = 0; k < p.dn; ++k) {
      const double v = V[i * p.dn + k];
#pragma unroll
      for (int j = 0; j < D; ++j) h[j] = fma(v, p.en.W1[k * D + j], h[j]);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) h[j] = act_fn<ACT>(h[j]);
    matvec<D, D>(h, p.en.W2, p.en.b2, x, D);
#pragma unroll
    for (int j = 0; j < D; ++j) X[i * D + j] = x[j];
    if (p.L > 0) {
      double o[D];
      matvec<D, D>(x, p.fm[0].W1, nullptr, o, D);
#pragma unroll
      for (int j = 0; j < D; ++j) PQ[i * 2 * D + j] = o[j];
      matvec<D, D>(x, p.fm[0].W1 + D * D, nullptr, o, D);
#pragma unroll
      for (int j = 0; j < D; ++j) PQ[i * 2 * D + D + j] = o[j];
    }
  }
}

// Layer t: message row-sum, node update, P'_t / Q'_t (edge pass) and next layer's P / Q.
template <int D, int ACT>
__global__ void k_node_layer(GnnP p, int t, int64_t n, const int32_t* __restrict__ offs,
                             const int32_t* __restrict__ cols, const double* __restrict__ ef,
                             double* X, const double* __restrict__ PQ, double* PQn,
                             double* EPQ) {
  const MlpP fm = p.fm[t], fv = p.fv[t], fe = p.fe[t];
  const double* c = fm.W1 + 2 * D * D;  // edge-feature row of W1m (d_edge == 1)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double S[D], pi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) { S[j] = 0.0; pi[j] = PQ[i * 2 * D + j] + fm.b1[j]; }
    const int32_t lo = offs[i], hi = offs[i + 1];
    for (int32_t k = lo; k < hi; ++k) {
      const double* qj = PQ + (int64_t)cols[k] * 2 * D + D;
      const double e = ef[k];
#pragma unroll
      for (int j = 0; j < D; ++j) S[j] += act_fn<ACT>(pi[j] + qj[j] + e * c[j]);
    }
    const double deg = (double)(hi - lo);
    double m[D];
    matvec<D, D>(S, fm.W2, nullptr, m, D);
#pragma unroll
    for (int j = 0; j < D; ++j) m[j] = fma(deg, fm.b2[j], m[j]);
    double u[D];
    matvec<D, D>(m, fv.W1, fv.b1, u, D);
#pragma unroll
    for (int j = 0; j < D; ++j) u[j] = act_fn<ACT>(u[j]);
    double x[D];
    matvec<D, D>(u, fv.W2, fv.b2, x, D);
#pragma unroll
    for (int j = 0; j < D; ++j) { x[j] = X[i * D + j] + x[j]; X[i * D + j] = x[j]; }
    double o[D];
    double* ep = EPQ + ((int64_t)t * n + i) * 2 * D;
    matvec<D, D>(x, fe.W1, nullptr, o, D);
#pragma unroll
    for (int j = 0; j < D; ++j) ep[j] = o[j];
    matvec<D, D>(x, fe.W1 + D * D, nullptr, o, D);
#pragma unroll
    for (int j = 0; j < D; ++j) ep[D + j] = o[j];
    if (t + 1 < p.L) {
      matvec<D, D>(x, p.fm[t + 1].W1, nullptr, o, D);
#pragma unroll
      for (int j = 0; j < D; ++j) PQn[i * 2 * D + j] = o[j];
      matvec<D, D>(x, p.fm[t + 1].W1 + D * D, nullptr, o, D);
#pragma unroll
      for (int j = 0; j < D; ++j) PQn[i * 2 * D + D + j] = o[j];
    }
  }
}

// Fused edge pass.  Edge-path weights are copied to shared memory:
//   [Ee1 D][be1 D][Ee2 DxD][be2 D] + L x ([We1c DxD][be1 D][We2 DxD][be2 D]) + [D1 DxD][bd1 D][D2 D][bd2 1]
template <int D>
__host__ __device__ constexpr int edge_smem_doubles(int L) {
  return (3 * D + D * D) + L * (2 * D * D + 2 * D) + (D * D + 2 * D + 1);
}

template <int D, int ACT>
__global__ void __launch_bounds__(128) k_edge_pass(GnnP p, int64_t nnz, const int32_t* __restrict__ rows,
                                                   const int32_t* __restrict__ cols,
                                                   const double* __restrict__ ef,
                                                   const double* __restrict__ EPQ, int64_t n,
                                                   double* __restrict__ g) {
  extern __shared__ double w[];
  const int L = p.L;
  {  // stage weights
    int o = 0;
    auto cp = [&](const double* src, int cnt) {
      for (int k = threadIdx.x; k < cnt; k += blockDim.x) w[o + k] = src[k];
      o += cnt;
    };
    cp(p.ee.W1, D); cp(p.ee.b1, D); cp(p.ee.W2, D * D); cp(p.ee.b2, D);
    for (int t = 0; t < L; ++t) {
      cp(p.fe[t].W1 + 2 * D * D, D * D); cp(p.fe[t].b1, D); cp(p.fe[t].W2, D * D); cp(p.fe[t].b2, D);
    }
    cp(p.dec.W1, D * D); cp(p.dec.b1, D); cp(p.dec.W2, D); cp(p.dec.b2, 1);
  }
  __syncthreads();
  const double* Ee1 = w;
  const double* eb1 = w + D;
  const double* Ee2 = w + 2 * D;
  const double* eb2 = w + 2 * D + D * D;
  const double* lay = w + 3 * D + D * D;
  const double* dec = lay + L * (2 * D * D + 2 * D);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double e = ef[k];
    const int64_t i = rows[k], j = cols[k];
    double h[D], a[D];
#pragma unroll
    for (int q = 0; q < D; ++q) a[q] = act_fn<ACT>(fma(e, Ee1[q], eb1[q]));
    matvec<D, D>(a, Ee2, eb2, h, D);
    for (int t = 0; t < L; ++t) {
      const double* W1c = lay + t * (2 * D * D + 2 * D);
      const double* b1 = W1c + D * D;
      const double* W2 = b1 + D;
      const double* b2 = W2 + D * D;
      const double* Pi = EPQ + ((int64_t)t * n + i) * 2 * D;
      const double* Qj = EPQ + ((int64_t)t * n + j) * 2 * D + D;
#pragma unroll
      for (int q = 0; q < D; ++q) a[q] = Pi[q] + Qj[q] + b1[q];
#pragma unroll
      for (int kk = 0; kk < D; ++kk) {
        const double v = h[kk];
#pragma unroll
        for (int q = 0; q < D; ++q) a[q] = fma(v, W1c[kk * D + q], a[q]);
      }
#pragma unroll
      for (int q = 0; q < D; ++q) a[q] = act_fn<ACT>(a[q]);
#pragma unroll
      for (int q = 0; q < D; ++q) h[q] += b2[q];
#pragma unroll
      for (int kk = 0; kk < D; ++kk) {
        const double v = a[kk];
#pragma unroll
        for (int q = 0; q < D; ++q) h[q] = fma(v, W2[kk * D + q], h[q]);
      }
    }
    matvec<D, D>(h, dec, dec + D * D, a, D);
    double out = dec[D * D + 2 * D];
#pragma unroll
    for (int q = 0; q < D; ++q) out = fma(act_fn<ACT>(a[q]), dec[D * D + D + q], out);
    g[k] = out;
  }
}

static int grid_for(int64_t n, int threads) {
  int64_t b = ceil_div(n > 0 ? n : 1, threads);
  return (int)(b > 148 * 16 ? 148 * 16 : b);
}

template <int D, int ACT>
int run_forward(const GnnP& p, int64_t n, int64_t nnz, const int32_t* offs, const int32_t* cols,
                const int32_t* rows, const double* V, const double* ef, double* g, double* X,
                double* PQa, double* PQb, double* EPQ, cudaStream_t s) {
  k_node_encode<D, ACT><<<grid_for(n, 128), 128, 0, s>>>(p, n, V, X, PQa);
  SG_LAUNCH_CHECK("k_node_encode");
  double* cur = PQa;
  double* nxt = PQb;
  for (int t = 0; t < p.L; ++t) {
    k_node_layer<D, ACT><<<grid_for(n, 128), 128, 0, s>>>(p, t, n, offs, cols, ef, X, cur, nxt, EPQ);
    SG_LAUNCH_CHECK("k_node_layer");
    double* tmp = cur; cur = nxt; nxt = tmp;
  }
  const size_t smem = edge_smem_doubles<D>(p.L) * sizeof(double);
  SG_CUDA(cudaFuncSetAttribute(k_edge_pass<D, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_edge_pass<D, ACT><<<grid_for(nnz, 128), 128, smem, s>>>(p, nnz, rows, cols, ef, EPQ, n, g);
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
