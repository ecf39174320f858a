// The reference's own noise predictor on device (fp64): predictor.py:133-166.
//
//   a0 = [x, time_embed(t)];  z_l = a_l W_l + b_l;  a_{l+1} = act(z_l) (hidden)
//
// W_l stays in the reference's (fan_in, fan_out) row-major layout, so a
// thread owning output column o streams W[:, o] with coalesced loads across
// the warp. Each layer is a deterministic two-phase split-K GEMV over the B
// lanes of a cycle (fixed reduction order, no atomics: every rank computes
// the same bits, which ParaStep's redundant warm-up relies on).

#include "common.cuh"

namespace ps {

constexpr int MLP_COLS = 64;   // output columns per block
constexpr int MLP_KGRP = 4;    // k-subgroups per block (threads = 64 x 4)
constexpr int MLP_KROWS = 64;  // K rows per block
constexpr int MLP_MAXB = PS_MAX_CYCLE;

struct MlpLayerArgs {
  const double* a;      // [B, K] activations (layer 0: unused, see x/temb)
  const double* x;      // layer 0: [B, data_dim]
  const double* temb;   // layer 0: table base
  int data_dim, embed_dim, layer0;
  int32_t ts[MLP_MAXB];
  const double* W;      // [K, N]
  int K, N, B, ks;
  double* partial;      // [ks, B, N]
};

__device__ __forceinline__ double act_in(const MlpLayerArgs& p, int b, int i) {
  if (!p.layer0) return p.a[(int64_t)b * p.K + i];
  if (i < p.data_dim) return p.x[(int64_t)b * p.data_dim + i];
  return p.temb[(int64_t)p.ts[b] * p.embed_dim + (i - p.data_dim)];
}

__global__ void __launch_bounds__(MLP_COLS * MLP_KGRP)
mlp_partial_kernel(const __grid_constant__ MlpLayerArgs p) {
  __shared__ double red[MLP_KGRP][MLP_MAXB][MLP_COLS];
  const int tx = threadIdx.x % MLP_COLS, ty = threadIdx.x / MLP_COLS;
  const int o = blockIdx.x * MLP_COLS + tx;
  const int k0 = blockIdx.y * MLP_KROWS;
  const int k1 = min(p.K, k0 + MLP_KROWS);
  double acc[MLP_MAXB];
#pragma unroll
  for (int b = 0; b < MLP_MAXB; ++b) acc[b] = 0.0;
  if (o < p.N) {
    for (int i = k0 + ty; i < k1; i += MLP_KGRP) {
      const double w = p.W[(int64_t)i * p.N + o];
#pragma unroll
      for (int b = 0; b < MLP_MAXB; ++b)
        if (b < p.B) acc[b] = fma(act_in(p, b, i), w, acc[b]);
    }
  }
#pragma unroll
  for (int b = 0; b < MLP_MAXB; ++b)
    if (b < p.B) red[ty][b][tx] = acc[b];
  __syncthreads();
  if (ty == 0 && o < p.N) {
    for (int b = 0; b < p.B; ++b) {
      double s = red[0][b][tx];
#pragma unroll
      for (int g = 1; g < MLP_KGRP; ++g) s += red[g][b][tx];
      p.partial[((int64_t)blockIdx.y * p.B + b) * p.N + o] = s;
    }
  }
}

// sign-split logistic of predictor.py:108-116
__device__ __forceinline__ double sigmoid_split(double z) {
  if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
  double e = exp(z);
  return e / (1.0 + e);
}

__global__ void mlp_finish_kernel(const double* partial, int ks, int B, int N, const double* bias,
                                  int act, double* out) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * N) return;
  int o = idx % N;
  double s = partial[idx];
  for (int k = 1; k < ks; ++k) s += partial[(int64_t)k * B * N + idx];
  double z = s + bias[o];
  double r;
  if (act < 0) r = z;                 // output layer: linear
  else if (act == 0) r = tanh(z);     // ACT_TANH
  else r = z * sigmoid_split(z);      // ACT_SILU
  out[idx] = r;
}

}  // namespace ps

using namespace ps;

extern "C" {

static int max_dim(const ps_mlp* m) {
  int d = 0;
  for (int l = 0; l <= m->n_layers; ++l) d = d > m->dims[l] ? d : m->dims[l];
  return d;
}

size_t ps_mlp_workspace_bytes(const ps_mlp* m, int B) {
  size_t part = 0;
  for (int l = 0; l < m->n_layers; ++l) {
    size_t ks = (m->dims[l] + MLP_KROWS - 1) / MLP_KROWS;
    size_t s = ks * (size_t)B * m->dims[l + 1];
    part = part > s ? part : s;
  }
  return (part + 2 * (size_t)B * max_dim(m)) * sizeof(double) + 256;
}

int ps_mlp_forward(const ps_mlp* m, const double* x, const int32_t* host_ts, int B, double* out,
                   void* workspace, void* cs) {
  PS_CHECK_ARG(m && m->n_layers >= 1 && m->n_layers <= 16, "bad MLP descriptor");
  PS_CHECK_ARG(B >= 1 && B <= MLP_MAXB, "batch must be in [1, 16]");
  PS_CHECK_ARG(m->dims[0] == m->data_dim + m->embed_dim, "dims[0] != data_dim + embed_dim");
  cudaStream_t st = as_stream(cs);
  size_t part = 0;
  for (int l = 0; l < m->n_layers; ++l) {
    size_t ks = (m->dims[l] + MLP_KROWS - 1) / MLP_KROWS;
    size_t s = ks * (size_t)B * m->dims[l + 1];
    part = part > s ? part : s;
  }
  double* partial = reinterpret_cast<double*>(workspace);
  double* buf[2] = {partial + part, partial + part + (size_t)B * max_dim(m)};
  const double* a = nullptr;
  for (int l = 0; l < m->n_layers; ++l) {
    MlpLayerArgs p{};
    p.a = a;
    p.x = x;
    p.temb = m->temb_table;
    p.data_dim = m->data_dim;
    p.embed_dim = m->embed_dim;
    p.layer0 = (l == 0);
    for (int b = 0; b < B; ++b) p.ts[b] = host_ts[b];
    p.W = m->W[l];
    p.K = m->dims[l];
    p.N = m->dims[l + 1];
    p.B = B;
    p.ks = (p.K + MLP_KROWS - 1) / MLP_KROWS;
    p.partial = partial;
    dim3 grid((p.N + MLP_COLS - 1) / MLP_COLS, p.ks);
    mlp_partial_kernel<<<grid, MLP_COLS * MLP_KGRP, 0, st>>>(p);
    int rc = check_launch("mlp_partial");
    if (rc) return rc;
    const bool last = (l == m->n_layers - 1);
    double* dst = last ? out : buf[l & 1];
    int total = B * p.N;
    mlp_finish_kernel<<<(total + 255) / 256, 256, 0, st>>>(partial, p.ks, B, p.N, m->b[l],
                                                           last ? -1 : m->activation, dst);
    rc = check_launch("mlp_finish");
    if (rc) return rc;
    a = dst;
  }
  return 0;
}

}  // extern "C"
