// Elementwise / normalisation / attention kernels of the DiT predictor.
// Architecture: paper_2505_14741_b200/spec.py. Residual stream fp32.
#pragma once

#include "common.cuh"

namespace ps {

struct DitGeom {
  int C, F, H, W, layout, p, D, L, gw, gh;
};

// latent flat index of channel c at frame f, pixel (y, x)
__device__ __forceinline__ int64_t latent_index(const DitGeom& g, int c, int f, int y, int x) {
  if (g.layout == 0) return (((int64_t)c * g.F + f) * g.H + y) * g.W + x;
  return (((int64_t)f * g.H + y) * g.W + x) * g.C + c;
}

// token l -> (f, hp, wp); patch feature k -> (c, ph, pw)
__device__ __forceinline__ int64_t patch_elem_index(const DitGeom& g, int l, int k) {
  const int per_f = g.gh * g.gw;
  const int f = l / per_f, r = l % per_f, hp = r / g.gw, wp = r % g.gw;
  const int pp = g.p * g.p;
  const int c = k / pp, q = k % pp, ph = q / g.p, pw = q % g.p;
  return latent_index(g, c, f, hp * g.p + ph, wp * g.p + pw);
}

__device__ __forceinline__ float silu_f(float v) { return v / (1.0f + expf(-v)); }

__device__ __forceinline__ float gelu_tanh_f(float v) {
  const float k0 = 0.7978845608028654f;  // sqrt(2/pi)
  return 0.5f * v * (1.0f + tanhf(k0 * (v + 0.044715f * (v * v * v))));
}

// ---------------------------------------------------------------- GEMV
// out[b, o] = act(sum_i in_b[i] W[i, o] + bias[o]); W (K, N) row-major.
// in_b = in + in_row[b] * in_stride (row index per lane, e.g. the step t for
// the frequency table). 32 columns x 8 k-groups per block, fixed-order
// smem reduction (deterministic).
constexpr int GV_COLS = 32, GV_KGRP = 8, GV_MAXB = 16;

struct GemvArgs {
  const float* in;
  int64_t in_stride;
  int32_t in_row[GV_MAXB];
  const float* W;
  const float* bias;
  float* out;
  int K, N, B, act;  // act: 0 none, 1 silu
};

static __global__ void __launch_bounds__(GV_COLS * GV_KGRP) gemv_kernel(const __grid_constant__ GemvArgs p) {
  __shared__ float red[GV_KGRP][GV_MAXB][GV_COLS + 1];
  const int tx = threadIdx.x % GV_COLS, ty = threadIdx.x / GV_COLS;
  const int o = blockIdx.x * GV_COLS + tx;
  float acc[GV_MAXB];
#pragma unroll
  for (int b = 0; b < GV_MAXB; ++b) acc[b] = 0.f;
  if (o < p.N) {
    for (int i = ty; i < p.K; i += GV_KGRP) {
      const float w = __ldg(p.W + (int64_t)i * p.N + o);
#pragma unroll
      for (int b = 0; b < GV_MAXB; ++b)
        if (b < p.B) acc[b] = fmaf(p.in[(int64_t)p.in_row[b] * p.in_stride + i], w, acc[b]);
    }
  }
#pragma unroll
  for (int b = 0; b < GV_MAXB; ++b)
    if (b < p.B) red[ty][b][tx] = acc[b];
  __syncthreads();
  for (int idx = threadIdx.x; idx < p.B * GV_COLS; idx += blockDim.x) {
    const int b = idx / GV_COLS, c = idx % GV_COLS, oo = blockIdx.x * GV_COLS + c;
    if (oo >= p.N) continue;
    float s = red[0][b][c];
#pragma unroll
    for (int g = 1; g < GV_KGRP; ++g) s += red[g][b][c];
    s += p.bias ? p.bias[oo] : 0.f;
    p.out[(int64_t)b * p.N + oo] = p.act == 1 ? silu_f(s) : s;
  }
}

// ---------------------------------------------------------------- patch embed
// h[b*L + l, d] = sum_k x_b[patch(l, k)] * Wpe[k, d] + bpe[d] + pos[l, d]
static __global__ void patch_embed_kernel(const float* __restrict__ x, int64_t n_latent, DitGeom g,
                                   int patch_dim, const float* __restrict__ Wpe,
                                   const float* __restrict__ bpe, const float* __restrict__ pos,
                                   float* __restrict__ h, int B) {
  extern __shared__ float patch_s[];  // patch_dim values of this token
  const int row = blockIdx.x;  // b*L + l
  const int b = row / g.L, l = row % g.L;
  for (int k = threadIdx.x; k < patch_dim; k += blockDim.x)
    patch_s[k] = x[(int64_t)b * n_latent + patch_elem_index(g, l, k)];
  __syncthreads();
  for (int d = threadIdx.x; d < g.D; d += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < patch_dim; ++k) s = fmaf(patch_s[k], Wpe[(int64_t)k * g.D + d], s);
    h[(int64_t)row * g.D + d] = s + bpe[d] + pos[(int64_t)l * g.D + d];
  }
}

// ---------------------------------------------------------------- LN + modulate
// a[row, :] = LN(h[row, :]) * (1 + scale_b) + shift_b ; one warp per row.
// Output formats: fp32 (out_f32), bf16 (out_bf16), or the tf32 hi/lo split
// (out_hi/out_lo) consumed by the 3xTF32 tensor-core GEMM.
struct LnModArgs {
  const float* h;
  int rows, D, L;
  const float* mod;  // per lane base of modulation vector block
  int64_t mod_stride;
  int shift_off, scale_off;
  float* out_f32;
  __nv_bfloat16* out_bf16;
  float* out_hi;
  float* out_lo;
};

__device__ __forceinline__ float tf32_hi(float v) {
  return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
}

__device__ __forceinline__ void store_act(const LnModArgs& p, int64_t idx, float v) {
  if (p.out_f32) p.out_f32[idx] = v;
  if (p.out_bf16) p.out_bf16[idx] = __float2bfloat16_rn(v);
  if (p.out_hi) {
    float hi = tf32_hi(v);
    p.out_hi[idx] = hi;
    p.out_lo[idx] = v - hi;
  }
}

static __global__ void ln_mod_kernel(const __grid_constant__ LnModArgs p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= p.rows) return;
  const float* hr = p.h + (int64_t)warp * p.D;
  float s = 0.f;
  for (int d = lane; d < p.D; d += 32) s += hr[d];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mu = s / p.D;
  float v = 0.f;
  for (int d = lane; d < p.D; d += 32) {
    float t = hr[d] - mu;
    v = fmaf(t, t, v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const float rstd = rsqrtf(v / p.D + 1e-6f);
  const int b = warp / p.L;
  const float* m = p.mod + (int64_t)b * p.mod_stride;
  for (int d = lane; d < p.D; d += 32) {
    float y = (hr[d] - mu) * rstd;
    y = fmaf(y, 1.f + m[p.scale_off + d], m[p.shift_off + d]);
    store_act(p, (int64_t)warp * p.D + d, y);
  }
}

// ---------------------------------------------------------------- attention
// Flash-style SIMT attention, fp32. qkv row m = [q(D) | k(D) | v(D)], head h
// in columns h*dh..; out row m = heads concatenated (spec.py). One block per
// (lane b, head, 64-query tile); 8 warps x 8 query rows; K/V tiles of 64 in
// smem; lane j owns keys j, j+32 for the scores, output dims d = lane+32u.
constexpr int AT_Q = 64, AT_K = 64, AT_WARPS = 8, AT_MAXU = 4;  // dh <= 128

struct AttnArgs {
  const float* qkv;
  int L, D, H, dh;
  float scale;
  float* out_f32;
  __nv_bfloat16* out_bf16;
  float* out_hi;
  float* out_lo;
};

static __global__ void __launch_bounds__(AT_WARPS * 32) attn_kernel(const __grid_constant__ AttnArgs p) {
  extern __shared__ float at_s[];
  const int dh = p.dh, ldk = dh + 1;
  float* Ks = at_s;                // [AT_K][ldk]
  float* Vs = Ks + AT_K * ldk;     // [AT_K][dh]
  float* Qs = Vs + AT_K * dh;      // [AT_Q][dh]
  const int qt = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (int64_t)b * p.L;
  const int ld = 3 * p.D;
  const int q0 = qt * AT_Q;
  for (int idx = threadIdx.x; idx < AT_Q * dh; idx += blockDim.x) {
    int r = idx / dh, d = idx % dh;
    int q = q0 + r;
    Qs[idx] = q < p.L ? p.qkv[(row0 + q) * ld + head * dh + d] * p.scale : 0.f;
  }
  float m_r[8], l_r[8], o_r[8][AT_MAXU];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    m_r[r] = -INFINITY;
    l_r[r] = 0.f;
#pragma unroll
    for (int u = 0; u < AT_MAXU; ++u) o_r[r][u] = 0.f;
  }
  const int nU = (dh + 31) / 32;
  for (int k0 = 0; k0 < p.L; k0 += AT_K) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < AT_K * dh; idx += blockDim.x) {
      int j = idx / dh, d = idx % dh;
      int kk = k0 + j;
      float kv = 0.f, vv = 0.f;
      if (kk < p.L) {
        const float* src = p.qkv + (row0 + kk) * ld + head * dh + d;
        kv = src[p.D];
        vv = src[2 * p.D];
      }
      Ks[j * ldk + d] = kv;
      Vs[j * dh + d] = vv;
    }
    __syncthreads();
    const int nk = min(AT_K, p.L - k0);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int qr = warp * 8 + r;
      const float* qrow = Qs + qr * dh;
      float s0 = 0.f, s1 = 0.f;
      const float* k0p = Ks + lane * ldk;
      const float* k1p = Ks + (lane + 32) * ldk;
      for (int d = 0; d < dh; ++d) {
        float qv = qrow[d];
        s0 = fmaf(qv, k0p[d], s0);
        s1 = fmaf(qv, k1p[d], s1);
      }
      if (lane >= nk) s0 = -INFINITY;
      if (lane + 32 >= nk) s1 = -INFINITY;
      float mx = fmaxf(s0, s1);
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float mnew = fmaxf(m_r[r], mx);
      const float corr = expf(m_r[r] - mnew);
      const float p0 = expf(s0 - mnew), p1 = expf(s1 - mnew);
      float ps = p0 + p1;
#pragma unroll
      for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      l_r[r] = l_r[r] * corr + ps;
      m_r[r] = mnew;
#pragma unroll
      for (int u = 0; u < AT_MAXU; ++u) o_r[r][u] *= corr;
      for (int j = 0; j < 32; ++j) {
        const float pa = __shfl_sync(0xffffffffu, p0, j);
        const float pb = __shfl_sync(0xffffffffu, p1, j);
#pragma unroll
        for (int u = 0; u < AT_MAXU; ++u) {
          const int d = lane + 32 * u;
          if (u < nU && d < dh)
            o_r[r][u] = fmaf(pa, Vs[j * dh + d], fmaf(pb, Vs[(j + 32) * dh + d], o_r[r][u]));
        }
      }
    }
  }
  LnModArgs st{};
  st.out_f32 = p.out_f32;
  st.out_bf16 = p.out_bf16;
  st.out_hi = p.out_hi;
  st.out_lo = p.out_lo;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int q = q0 + warp * 8 + r;
    if (q >= p.L) continue;
    const float inv = 1.f / l_r[r];
#pragma unroll
    for (int u = 0; u < AT_MAXU; ++u) {
      const int d = lane + 32 * u;
      if (u < nU && d < dh) store_act(st, (row0 + q) * p.D + head * dh + d, o_r[r][u] * inv);
    }
  }
}

}  // namespace ps
