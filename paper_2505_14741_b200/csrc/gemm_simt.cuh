// SIMT fp32 GEMM with the DiT epilogues. This is the fp32 baseline and the
// on-device cross-check for the tcgen05 kernels (gemm_tc.cuh); the fast
// path uses tensor cores.
//   C[M, N] = A[M, K] (row-major) x W[K, N] (row-major, reference layout)
#pragma once

#include "dit_kernels.cuh"

namespace ps {

enum EpiMode { EPI_STORE = 0, EPI_GELU = 1, EPI_RESID = 2, EPI_UNPATCH = 3 };

struct Epi {
  int mode;
  const float* bias;
  // EPI_STORE: out[M, N] fp32; EPI_GELU: act formats
  float* out;
  __nv_bfloat16* out_bf16;
  float* out_hi;
  float* out_lo;
  // EPI_RESID: resid[m, n] += gate[b(m) * gate_stride + n] * (acc + bias)
  float* resid;
  const float* gate;
  int64_t gate_stride;
  int L;  // rows per lane
  // EPI_UNPATCH: eps[b * n_latent + latent(token, feature)] = acc + bias
  DitGeom g;
  float* eps;
  int64_t n_latent;
};

__device__ __forceinline__ void epi_store(const Epi& e, int m, int n, int N, float acc) {
  const float v = acc + (e.bias ? e.bias[n] : 0.f);
  const int64_t idx = (int64_t)m * N + n;
  switch (e.mode) {
    case EPI_STORE:
      e.out[idx] = v;
      break;
    case EPI_GELU: {
      const float g = gelu_tanh_f(v);
      if (e.out) e.out[idx] = g;
      if (e.out_bf16) e.out_bf16[idx] = __float2bfloat16_rn(g);
      if (e.out_hi) {
        const float hi = tf32_hi(g);
        e.out_hi[idx] = hi;
        e.out_lo[idx] = g - hi;
      }
      break;
    }
    case EPI_RESID: {
      const int b = m / e.L;
      e.resid[idx] = fmaf(e.gate[(int64_t)b * e.gate_stride + n], v, e.resid[idx]);
      break;
    }
    case EPI_UNPATCH: {
      const int b = m / e.g.L, l = m % e.g.L;
      e.eps[(int64_t)b * e.n_latent + patch_elem_index(e.g, l, n)] = v;
      break;
    }
  }
}

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

static __global__ void __launch_bounds__(256) gemm_simt_kernel(const float* __restrict__ A,
                                                       const float* __restrict__ W, int M, int N,
                                                       int K, const __grid_constant__ Epi e) {
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += SG_BK) {
    for (int idx = threadIdx.x; idx < SG_BM * SG_BK; idx += 256) {
      const int r = idx / SG_BK, kk = idx % SG_BK;
      const int gm = m0 + r, gk = k0 + kk;
      As[kk][r] = (gm < M && gk < K) ? A[(int64_t)gm * K + gk] : 0.f;
    }
    for (int idx = threadIdx.x; idx < SG_BK * SG_BN; idx += 256) {
      const int kk = idx / SG_BN, c = idx % SG_BN;
      const int gk = k0 + kk, gn = n0 + c;
      Bs[kk][c] = (gk < K && gn < N) ? W[(int64_t)gk * N + gn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) epi_store(e, m, n, N, acc[i][j]);
    }
}

}  // namespace ps
