// SIMT fp32 GEMM with the DiT epilogues. This is the fp32 baseline and the
// on-device cross-check for the tcgen05 kernels (gemm_tc.cuh); the fast
// path uses tensor cores.
//   C[M, N] = A[M, K] (row-major) x W[K, N] (row-major, reference layout)
#pragma once

#include "dit_kernels.cuh"

namespace ps {

enum EpiMode { EPI_STORE = 0, EPI_GELU = 1, EPI_RESID = 2, EPI_UNPATCH = 3, EPI_ADD = 4, EPI_NCHW = 5 };

struct Epi {
  int mode;
  const float* bias;
  // EPI_STORE: out[M, N] fp32 and/or out_bf16; EPI_GELU: act formats
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
  // EPI_ADD (U-Net): y = act(acc + bias + vec[b(m) * vec_stride + n] + resid[m, n]),
  // each term optional; y -> out (fp32) and/or out_bf16. b(m) = m / L.
  const float* vec;
  int64_t vec_stride;
  int act;  // 1 = GELU-tanh
  // EPI_NCHW: eps[b * n_latent + n * hw + p] = acc + bias, m = b * hw + p
  int hw;
  // per-lane rows of gate / vec: lane b reads row lane_row[b] (a per-run
  // conditioning table indexed by t) when use_rows, else row b
  int use_rows;
  int32_t lane_row[16];
  // EPI_STORE bf16 into a head-padded operand: column n = (w*H + h)*pad_dh + d
  // goes to (w*H + h)*pad_DH + d of a row of N/pad_dh*pad_DH (0 = dense)
  int pad_dh, pad_DH;
  // text rows (spec.py text_tokens): rows with m % L < txt are text tokens;
  // EPI_RESID reads their gate txt_delta floats further along the row
  // (expert adaLN); EPI_UNPATCH skips them (L = txt + video tokens there)
  int txt;
  int64_t txt_delta;
  // EPI_STORE of the QKV GEMM: 3D RoPE on the q and k columns (n < 2 * rope_D)
  // of video rows, interleaved pairs; rope[(v * rope_dh / 2 + i) * 2 + {0, 1}]
  // = (cos, sin) of pair i of video token v
  const float* rope;
  int rope_dh, rope_D;
};

// gate row of EPI_RESID for row m (text rows: the text half of the adaLN block)
__device__ __forceinline__ const float* gate_row(const Epi& e, int m);

// RoPE on 4 consecutive columns n..n+3 (n % 4 == 0) of row m, in place
__device__ __forceinline__ void epi_rope4(const Epi& e, int m, int n, float* x) {
  if (!e.rope || n >= 2 * e.rope_D) return;
  const int v = m % e.L - e.txt;
  if (v < 0) return;
  const int i0 = (n % e.rope_dh) >> 1;
  const float4 cs =
      *reinterpret_cast<const float4*>(e.rope + ((int64_t)v * (e.rope_dh >> 1) + i0) * 2);
  const float a0 = x[0], a1 = x[1], a2 = x[2], a3 = x[3];
  x[0] = a0 * cs.x - a1 * cs.y;
  x[1] = a1 * cs.x + a0 * cs.y;
  x[2] = a2 * cs.z - a3 * cs.w;
  x[3] = a3 * cs.z + a2 * cs.w;
}

__device__ __forceinline__ int64_t lane_row(const Epi& e, int m) {
  const int b = m / e.L;
  return e.use_rows ? e.lane_row[b] : b;
}

__device__ __forceinline__ const float* gate_row(const Epi& e, int m) {
  const int64_t t = (e.txt && m % e.L < e.txt) ? e.txt_delta : 0;
  return e.gate + lane_row(e, m) * e.gate_stride + t;
}

__device__ __forceinline__ int64_t padded_index(const Epi& e, int m, int n, int N) {
  return (int64_t)m * (N / e.pad_dh * e.pad_DH) + (n / e.pad_dh) * e.pad_DH + n % e.pad_dh;
}

// GELU of an epilogue: MUFU tanh when the only output is bf16, the accurate
// tanhf whenever an fp32 (or tf32 hi/lo) value leaves the kernel
__device__ __forceinline__ float epi_gelu(const Epi& e, float v) {
  return (e.out_bf16 && !e.out && !e.out_hi) ? gelu_tanh_fast(v) : gelu_tanh_f(v);
}

__device__ __forceinline__ float epi_add_val(const Epi& e, int m, int n, int64_t idx, float v) {
  if (e.vec) v += e.vec[lane_row(e, m) * e.vec_stride + n];
  if (e.resid) v += e.resid[idx];
  return e.act ? epi_gelu(e, v) : v;
}

__device__ __forceinline__ void epi_store(const Epi& e, int m, int n, int N, float acc) {
  const float v = acc + (e.bias ? e.bias[n] : 0.f);
  const int64_t idx = (int64_t)m * N + n;
  switch (e.mode) {
    case EPI_STORE:
      if (e.out) e.out[idx] = v;
      if (e.out_bf16) e.out_bf16[e.pad_DH ? padded_index(e, m, n, N) : idx] = __float2bfloat16_rn(v);
      break;
    case EPI_GELU: {
      const float g = epi_gelu(e, v);
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
      e.resid[idx] = fmaf(gate_row(e, m)[n], v, e.resid[idx]);
      break;
    }
    case EPI_UNPATCH: {  // rows of a lane: txt text rows (skipped), then g.L video tokens
      const int Lt = e.g.L + e.txt;
      const int b = m / Lt, l = m % Lt - e.txt;
      if (l >= 0) e.eps[(int64_t)b * e.n_latent + patch_elem_index(e.g, l, n)] = v;
      break;
    }
    case EPI_ADD: {
      const float y = epi_add_val(e, m, n, idx, v);
      if (e.out) e.out[idx] = y;
      if (e.out_bf16) e.out_bf16[idx] = __float2bfloat16_rn(y);
      break;
    }
    case EPI_NCHW: {
      const int b = m / e.hw, px = m % e.hw;
      e.eps[(int64_t)b * e.n_latent + (int64_t)n * e.hw + px] = v;
      break;
    }
  }
}

// 16 consecutive columns n..n+15 of one row (tensor-core epilogue): 16-byte
// vector loads/stores when the row segment is full and aligned.
__device__ __forceinline__ void epi_store16(const Epi& e, int m, int n, int N, const float* v) {
  const bool vec = (n + 16 <= N) && ((N & 7) == 0) && e.mode != EPI_UNPATCH &&
                   e.mode != EPI_NCHW && (!e.pad_DH || e.mode == EPI_STORE);
  if (!vec) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (n + j < N) epi_store(e, m, n + j, N, v[j]);
    return;
  }
  const int64_t base = (int64_t)m * N + n;
  float x[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 bb = e.bias ? *reinterpret_cast<const float4*>(e.bias + n + 4 * q)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    x[4 * q] = v[4 * q] + bb.x;
    x[4 * q + 1] = v[4 * q + 1] + bb.y;
    x[4 * q + 2] = v[4 * q + 2] + bb.z;
    x[4 * q + 3] = v[4 * q + 3] + bb.w;
  }
  if (e.mode == EPI_STORE) {
#pragma unroll
    for (int q = 0; q < 4; ++q) epi_rope4(e, m, n + 4 * q, x + 4 * q);
    if (e.out)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(e.out + base + 4 * q) =
            make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
    if (e.out_bf16) {  // bf16 copy (the tcgen05 attention's Q/K/V operand)
      uint32_t u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * q], x[2 * q + 1]);
        u[q] = *reinterpret_cast<uint32_t*>(&h2);
      }
      // head-padded operand: each 8-column group lies inside one head (dh % 8 == 0)
      const int64_t i0 = e.pad_DH ? padded_index(e, m, n, N) : base;
      const int64_t i1 = e.pad_DH ? padded_index(e, m, n + 8, N) : base + 8;
      *reinterpret_cast<uint4*>(e.out_bf16 + i0) = make_uint4(u[0], u[1], u[2], u[3]);
      *reinterpret_cast<uint4*>(e.out_bf16 + i1) = make_uint4(u[4], u[5], u[6], u[7]);
    }
  } else if (e.mode == EPI_GELU) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = epi_gelu(e, x[j]);
    if (e.out)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(e.out + base + 4 * q) =
            make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
    if (e.out_bf16) {
      uint32_t u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * q], x[2 * q + 1]);
        u[q] = *reinterpret_cast<uint32_t*>(&h2);
      }
      *reinterpret_cast<uint4*>(e.out_bf16 + base) = make_uint4(u[0], u[1], u[2], u[3]);
      *reinterpret_cast<uint4*>(e.out_bf16 + base + 8) = make_uint4(u[4], u[5], u[6], u[7]);
    }
    if (e.out_hi) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 hi = make_float4(tf32_hi(x[4 * q]), tf32_hi(x[4 * q + 1]), tf32_hi(x[4 * q + 2]),
                                tf32_hi(x[4 * q + 3]));
        *reinterpret_cast<float4*>(e.out_hi + base + 4 * q) = hi;
        *reinterpret_cast<float4*>(e.out_lo + base + 4 * q) =
            make_float4(x[4 * q] - hi.x, x[4 * q + 1] - hi.y, x[4 * q + 2] - hi.z,
                        x[4 * q + 3] - hi.w);
      }
    }
  } else if (e.mode == EPI_ADD) {
    if (e.vec) {
      const float* vv = e.vec + lane_row(e, m) * e.vec_stride + n;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 a = *reinterpret_cast<const float4*>(vv + 4 * q);
        x[4 * q] += a.x; x[4 * q + 1] += a.y; x[4 * q + 2] += a.z; x[4 * q + 3] += a.w;
      }
    }
    if (e.resid) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 a = *reinterpret_cast<const float4*>(e.resid + base + 4 * q);
        x[4 * q] += a.x; x[4 * q + 1] += a.y; x[4 * q + 2] += a.z; x[4 * q + 3] += a.w;
      }
    }
    if (e.act)
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = epi_gelu(e, x[j]);
    if (e.out)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(e.out + base + 4 * q) =
            make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
    if (e.out_bf16) {
      uint32_t u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(x[2 * q], x[2 * q + 1]);
        u[q] = *reinterpret_cast<uint32_t*>(&h2);
      }
      *reinterpret_cast<uint4*>(e.out_bf16 + base) = make_uint4(u[0], u[1], u[2], u[3]);
      *reinterpret_cast<uint4*>(e.out_bf16 + base + 8) = make_uint4(u[4], u[5], u[6], u[7]);
    }
  } else {  // EPI_RESID
    const float* g = gate_row(e, m) + n;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4 r = *reinterpret_cast<const float4*>(e.resid + base + 4 * q);
      const float4 gg = *reinterpret_cast<const float4*>(g + 4 * q);
      r.x = fmaf(gg.x, x[4 * q], r.x);
      r.y = fmaf(gg.y, x[4 * q + 1], r.y);
      r.z = fmaf(gg.z, x[4 * q + 2], r.z);
      r.w = fmaf(gg.w, x[4 * q + 3], r.w);
      *reinterpret_cast<float4*>(e.resid + base + 4 * q) = r;
    }
  }
}

// 4 consecutive columns n..n+3 of one row (the split-K reduction's grain)
__device__ __forceinline__ void epi_store4(const Epi& e, int m, int n, int N, const float* v) {
  const bool vec = (n + 4 <= N) && ((N & 3) == 0) && e.mode != EPI_UNPATCH &&
                   e.mode != EPI_NCHW && (!e.pad_DH || e.mode == EPI_STORE);
  if (!vec) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (n + j < N) epi_store(e, m, n + j, N, v[j]);
    return;
  }
  const int64_t base = (int64_t)m * N + n;
  const float4 bb = e.bias ? *reinterpret_cast<const float4*>(e.bias + n)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
  float x[4] = {v[0] + bb.x, v[1] + bb.y, v[2] + bb.z, v[3] + bb.w};
  auto st_f32 = [&](float* out) {
    *reinterpret_cast<float4*>(out + base) = make_float4(x[0], x[1], x[2], x[3]);
  };
  auto st_bf16 = [&](__nv_bfloat16* out) {
    __nv_bfloat162 a = __floats2bfloat162_rn(x[0], x[1]), c = __floats2bfloat162_rn(x[2], x[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&c);
    *reinterpret_cast<uint2*>(out + (e.pad_DH ? padded_index(e, m, n, N) : base)) = u;
  };
  if (e.mode == EPI_STORE) {
    epi_rope4(e, m, n, x);
    if (e.out) st_f32(e.out);
    if (e.out_bf16) st_bf16(e.out_bf16);
  } else if (e.mode == EPI_GELU) {
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = epi_gelu(e, x[j]);
    if (e.out) st_f32(e.out);
    if (e.out_bf16) st_bf16(e.out_bf16);
    if (e.out_hi) {
      const float4 hi = make_float4(tf32_hi(x[0]), tf32_hi(x[1]), tf32_hi(x[2]), tf32_hi(x[3]));
      *reinterpret_cast<float4*>(e.out_hi + base) = hi;
      *reinterpret_cast<float4*>(e.out_lo + base) =
          make_float4(x[0] - hi.x, x[1] - hi.y, x[2] - hi.z, x[3] - hi.w);
    }
  } else if (e.mode == EPI_ADD) {
    if (e.vec) {
      const float4 a = *reinterpret_cast<const float4*>(e.vec + lane_row(e, m) * e.vec_stride + n);
      x[0] += a.x; x[1] += a.y; x[2] += a.z; x[3] += a.w;
    }
    if (e.resid) {
      const float4 a = *reinterpret_cast<const float4*>(e.resid + base);
      x[0] += a.x; x[1] += a.y; x[2] += a.z; x[3] += a.w;
    }
    if (e.act)
#pragma unroll
      for (int j = 0; j < 4; ++j) x[j] = epi_gelu(e, x[j]);
    if (e.out) st_f32(e.out);
    if (e.out_bf16) st_bf16(e.out_bf16);
  } else {  // EPI_RESID
    const float4 g = *reinterpret_cast<const float4*>(gate_row(e, m) + n);
    float4 r = *reinterpret_cast<const float4*>(e.resid + base);
    r.x = fmaf(g.x, x[0], r.x);
    r.y = fmaf(g.y, x[1], r.y);
    r.z = fmaf(g.z, x[2], r.z);
    r.w = fmaf(g.w, x[3], r.w);
    *reinterpret_cast<float4*>(e.resid + base) = r;
  }
}

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

static __global__ void __launch_bounds__(256) gemm_simt_kernel(const float* __restrict__ A,
                                                       const float* __restrict__ W, int M, int N,
                                                       int K, const __grid_constant__ Epi e) {
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  pdl_wait_and_release();
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
