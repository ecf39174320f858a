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

// The same GELU with the MUFU tanh (tanh.approx, rel. error ~2^-11): for
// outputs that are rounded to bf16 (2^-9) anyway. The accurate tanhf costs
// ~15% of a large-M bf16 GEMM whose epilogue applies it (CogVideoX fc1).
__device__ __forceinline__ float gelu_tanh_fast(float v) {
  const float k0 = 0.7978845608028654f;
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(k0 * (v + 0.044715f * (v * v * v))));
  return 0.5f * v * (1.0f + t);
}

// ---------------------------------------------------------------- GEMV
// out[b, o] = act(sum_i in_b[i] W[i, o] + bias[o]); W (K, N) row-major, fp32
// or bf16. in_b = in + in_row[b] * in_stride (e.g. the step t selects a row
// of the frequency table). HBM-bound on W: each lane streams 16 B of a row
// (4 fp32 / 8 bf16 columns), 8 warps split K, the B inputs are staged in
// smem, and the 8 partial sums are reduced in a fixed order (deterministic).
constexpr int GV_WARPS = 8, GV_MAXB = 16;

struct GemvArgs {
  const float* in;
  int64_t in_stride;
  int32_t in_row[GV_MAXB];
  const void* W;
  const float* bias;
  float* out;
  int K, N, B, act;  // act: 0 none, 1 silu
};

template <typename TW> struct GvLoad;
template <> struct GvLoad<float> {
  static constexpr int C = 4;
  static __device__ __forceinline__ void ld(const void* W, int64_t idx, float* w) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(W) + idx));
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  }
};
template <> struct GvLoad<__nv_bfloat16> {
  static constexpr int C = 8;
  static __device__ __forceinline__ void ld(const void* W, int64_t idx, float* w) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(
        reinterpret_cast<const __nv_bfloat16*>(W) + idx));
    const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      w[2 * q] = __uint_as_float(u[q] << 16);
      w[2 * q + 1] = __uint_as_float(u[q] & 0xFFFF0000u);
    }
  }
};

template <typename TW, int MAXB>
__global__ void __launch_bounds__(GV_WARPS * 32) gemv_kernel(const __grid_constant__ GemvArgs p) {
  constexpr int C = GvLoad<TW>::C;
  pdl_wait_and_release();
  extern __shared__ float gv_smem[];
  float* xin = gv_smem;                          // [B][K]
  float* red = gv_smem + (size_t)p.B * p.K;      // [GV_WARPS][B][32*C]
  for (int idx = threadIdx.x; idx < p.B * p.K; idx += blockDim.x) {
    const int b = idx / p.K, i = idx % p.K;
    xin[idx] = p.in[(int64_t)p.in_row[b] * p.in_stride + i];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col0 = blockIdx.x * 32 * C + lane * C;
  float acc[MAXB][C];
#pragma unroll
  for (int b = 0; b < MAXB; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[b][c] = 0.f;
  if (col0 < p.N) {
#pragma unroll 4
    for (int i = warp; i < p.K; i += GV_WARPS) {
      float w[C];
      GvLoad<TW>::ld(p.W, (int64_t)i * p.N + col0, w);
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        if (b < p.B) {
          const float xv = xin[b * p.K + i];
#pragma unroll
          for (int c = 0; c < C; ++c) acc[b][c] = fmaf(xv, w[c], acc[b][c]);
        }
      }
    }
  }
#pragma unroll
  for (int b = 0; b < MAXB; ++b)
    if (b < p.B)
#pragma unroll
      for (int c = 0; c < C; ++c) red[((size_t)warp * p.B + b) * (32 * C) + lane * C + c] = acc[b][c];
  __syncthreads();
  for (int idx = threadIdx.x; idx < p.B * 32 * C; idx += blockDim.x) {
    const int b = idx / (32 * C), cc = idx % (32 * C);
    const int o = blockIdx.x * 32 * C + cc;
    if (o >= p.N) continue;
    float s = 0.f;
#pragma unroll
    for (int g = 0; g < GV_WARPS; ++g) s += red[((size_t)g * p.B + b) * (32 * C) + cc];
    s += p.bias ? p.bias[o] : 0.f;
    p.out[(int64_t)b * p.N + o] = p.act == 1 ? silu_f(s) : s;
  }
}

template <typename TW>
static size_t gemv_smem(int B, int K) {
  return ((size_t)B * K + (size_t)GV_WARPS * B * 32 * GvLoad<TW>::C) * sizeof(float);
}

// ---------------------------------------------------------------- patch embed
// h[b*L + l, d] = sum_k x_b[patch(l, k)] * Wpe[k, d] + bpe[d] + pos[l, d]
// h rows of one lane: `txt` text rows copied from the fixed text states
// (spec.py), then the patch embedding of each video token (+ the additive
// position table when there is one; RoPE specs pass pos = null)
static __global__ void patch_embed_kernel(const float* __restrict__ x, int64_t n_latent, DitGeom g,
                                   int patch_dim, const float* __restrict__ Wpe,
                                   const float* __restrict__ bpe, const float* __restrict__ pos,
                                   float* __restrict__ h, int B, int txt,
                                   const float* __restrict__ text) {
  extern __shared__ float patch_s[];  // patch_dim values of this token
  pdl_wait_and_release();
  const int Lt = g.L + txt;
  const int row = blockIdx.x;  // b*Lt + l
  const int b = row / Lt, l = row % Lt - txt;
  if (l < 0) {
    for (int d = threadIdx.x; d < g.D; d += blockDim.x)
      h[(int64_t)row * g.D + d] = text[(int64_t)(l + txt) * g.D + d];
    return;
  }
  for (int k = threadIdx.x; k < patch_dim; k += blockDim.x)
    patch_s[k] = x[(int64_t)b * n_latent + patch_elem_index(g, l, k)];
  __syncthreads();
  for (int d = threadIdx.x; d < g.D; d += blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < patch_dim; ++k) s = fmaf(patch_s[k], Wpe[(int64_t)k * g.D + d], s);
    h[(int64_t)row * g.D + d] = s + bpe[d] + (pos ? pos[(int64_t)l * g.D + d] : 0.f);
  }
}

// host wrappers (one launch; B rows of `in` selected by `rows`)
template <typename TW, int MAXB>
static inline void gemv_launch(const GemvArgs& p, cudaStream_t st) {
  constexpr int C = GvLoad<TW>::C;
  const size_t smem = gemv_smem<TW>(p.B, p.K);
  launch_pdl(gemv_kernel<TW, MAXB>, dim3((p.N + 32 * C - 1) / (32 * C)), dim3(GV_WARPS * 32), smem,
             st, p);
}

template <typename TW>
static inline void gemv_set_attr() {
  cudaFuncSetAttribute(gemv_kernel<TW, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  cudaFuncSetAttribute(gemv_kernel<TW, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  cudaFuncSetAttribute(gemv_kernel<TW, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
  cudaFuncSetAttribute(gemv_kernel<TW, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10);
}

// W is fp32 or bf16 (wbf16), (K, N) row-major, N % (4|8) == 0
static inline int gemv(const float* in, int64_t in_stride, const int32_t* rows, const void* W, bool wbf16,
                const float* bias, float* out, int K, int N, int B, int act, cudaStream_t st) {
  GemvArgs p{};
  p.in = in;
  p.in_stride = in_stride;
  for (int b = 0; b < B; ++b) p.in_row[b] = rows ? rows[b] : b;
  p.W = W;
  p.bias = bias;
  p.out = out;
  p.K = K;
  p.N = N;
  p.B = B;
  p.act = act;
  if (wbf16) {
    if (B <= 1) gemv_launch<__nv_bfloat16, 1>(p, st);
    else if (B <= 4) gemv_launch<__nv_bfloat16, 4>(p, st);
    else if (B <= 8) gemv_launch<__nv_bfloat16, 8>(p, st);
    else gemv_launch<__nv_bfloat16, 16>(p, st);
  } else {
    if (B <= 1) gemv_launch<float, 1>(p, st);
    else if (B <= 4) gemv_launch<float, 4>(p, st);
    else if (B <= 8) gemv_launch<float, 8>(p, st);
    else gemv_launch<float, 16>(p, st);
  }
  return check_launch("gemv");
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
  int use_rows;              // lane b reads mod row mod_row[b] (else row b)
  int32_t mod_row[GV_MAXB];
  int shift_off, scale_off;
  int txt;        // text rows per lane (row % L < txt) read their shift / scale
  int txt_delta;  // this many floats further along the adaLN row (expert adaLN)
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

// one warp per row, the row held in registers (D <= 2048, D % 4 == 0):
// single read of h, two-pass mean/variance from registers, vector stores.
constexpr int LN_MAXV = 16;  // float4 per lane

__device__ __forceinline__ void store_act4(const LnModArgs& p, int64_t idx, float4 v) {
  if (p.out_f32) *reinterpret_cast<float4*>(p.out_f32 + idx) = v;
  if (p.out_bf16) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p.out_bf16 + idx) = u;
  }
  if (p.out_hi) {
    float4 hi = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
    *reinterpret_cast<float4*>(p.out_hi + idx) = hi;
    *reinterpret_cast<float4*>(p.out_lo + idx) =
        make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
  }
}

static __global__ void __launch_bounds__(256) ln_mod_kernel(const __grid_constant__ LnModArgs p) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int D4 = p.D >> 2;
  if (row < p.rows) {
    // the adaLN rows come from kernels that completed before the predecessor
    // (PDL chain): pull this lane's shift / scale into L1 while the
    // predecessor finishes
    const int b = row / p.L;
    const int64_t mrow = p.use_rows ? p.mod_row[b] : b;
    const int td = (p.txt && row % p.L < p.txt) ? p.txt_delta : 0;
    const float* base = p.mod + mrow * p.mod_stride + td;
    for (int i = lane; i < D4; i += 32) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(base + p.shift_off + 4 * i));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(base + p.scale_off + 4 * i));
    }
  }
  pdl_wait_and_release();
  if (row >= p.rows) return;
  const float4* hr = reinterpret_cast<const float4*>(p.h + (int64_t)row * p.D);
  float4 v[LN_MAXV];
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < LN_MAXV; ++u) {
    const int i = lane + 32 * u;
    v[u] = i < D4 ? hr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[u].x + v[u].y) + (v[u].z + v[u].w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mu = s / p.D;
  float q = 0.f;
#pragma unroll
  for (int u = 0; u < LN_MAXV; ++u) {
    if (lane + 32 * u < D4) {
      const float a = v[u].x - mu, b = v[u].y - mu, c = v[u].z - mu, d = v[u].w - mu;
      q = fmaf(a, a, fmaf(b, b, fmaf(c, c, fmaf(d, d, q))));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / p.D + 1e-6f);
  const int b = row / p.L;
  const int64_t mrow = p.use_rows ? p.mod_row[b] : b;
  const int td = (p.txt && row % p.L < p.txt) ? p.txt_delta : 0;
  const float4* sh =
      reinterpret_cast<const float4*>(p.mod + mrow * p.mod_stride + p.shift_off + td);
  const float4* sc =
      reinterpret_cast<const float4*>(p.mod + mrow * p.mod_stride + p.scale_off + td);
#pragma unroll
  for (int u = 0; u < LN_MAXV; ++u) {
    const int i = lane + 32 * u;
    if (i < D4) {
      const float4 a = sh[i], c = sc[i];
      float4 y;
      y.x = fmaf((v[u].x - mu) * rstd, 1.f + c.x, a.x);
      y.y = fmaf((v[u].y - mu) * rstd, 1.f + c.y, a.y);
      y.z = fmaf((v[u].z - mu) * rstd, 1.f + c.z, a.z);
      y.w = fmaf((v[u].w - mu) * rstd, 1.f + c.w, a.w);
      store_act4(p, (int64_t)row * p.D + 4 * i, y);
    }
  }
}

// ---------------------------------------------------------------- final layer
// The DiT's final layer as ONE warp-per-row kernel for small row counts:
// LayerNorm (two-pass, registers) + the final adaLN modulate + the linear
// projection to the P patch features (fp32 FMA, W in the reference layout
// (D, P)) + bias + the unpatchify scatter into eps. Replaces LN-modulate +
// a split-K tensor-core GEMM of N = P (16 for the 4-channel latents) - two
// launches and an A round trip - where the GEMM is tiny. Text rows (m % L <
// txt) carry no latent output and are skipped.
constexpr int FL_MAXP = 64;  // P <= 64 (4 and 16 channels x 2x2 patches)

struct FinalArgs {
  LnModArgs ln;  // h, rows, D, L, mod rows, shift/scale offsets (txt rows skipped)
  const float* W;  // [D][P] fp32
  const float* bias;  // [P]
  int P;
  DitGeom g;
  float* eps;
  int64_t n_latent;
};

template <int P>
static __global__ void __launch_bounds__(256) final_layer_kernel(const __grid_constant__ FinalArgs f) {
  const LnModArgs& p = f.ln;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int D4 = p.D >> 2;
  if (row < p.rows) {  // adaLN rows: written >= 2 kernels earlier (see ln_mod_kernel)
    const int b = row / p.L;
    const int64_t mrow = p.use_rows ? p.mod_row[b] : b;
    const float* base = p.mod + mrow * p.mod_stride;
    for (int i = lane; i < D4; i += 32) {
      asm volatile("prefetch.global.L1 [%0];" ::"l"(base + p.shift_off + 4 * i));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(base + p.scale_off + 4 * i));
    }
  }
  pdl_wait_and_release();
  if (row >= p.rows) return;
  const int b = row / p.L, l = row % p.L - p.txt;
  if (l < 0) return;  // text row
  const float4* hr = reinterpret_cast<const float4*>(p.h + (int64_t)row * p.D);
  float4 v[LN_MAXV];
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < LN_MAXV; ++u) {
    const int i = lane + 32 * u;
    v[u] = i < D4 ? hr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[u].x + v[u].y) + (v[u].z + v[u].w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mu = s / p.D;
  float q = 0.f;
#pragma unroll
  for (int u = 0; u < LN_MAXV; ++u) {
    if (lane + 32 * u < D4) {
      const float a = v[u].x - mu, c = v[u].y - mu, d = v[u].z - mu, e = v[u].w - mu;
      q = fmaf(a, a, fmaf(c, c, fmaf(d, d, fmaf(e, e, q))));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / p.D + 1e-6f);
  const int64_t mrow = p.use_rows ? p.mod_row[b] : b;
  const float4* sh = reinterpret_cast<const float4*>(p.mod + mrow * p.mod_stride + p.shift_off);
  const float4* sc = reinterpret_cast<const float4*>(p.mod + mrow * p.mod_stride + p.scale_off);
  // this lane's k = 4 (lane + 32 u) + j: partial dot products for all P outputs
  float acc[P];
#pragma unroll
  for (int j = 0; j < P; ++j) acc[j] = 0.f;
#pragma unroll
  for (int u = 0; u < LN_MAXV; ++u) {
    const int i = lane + 32 * u;
    if (i >= D4) break;
    const float4 a = sh[i], c = sc[i];
    const float y[4] = {fmaf((v[u].x - mu) * rstd, 1.f + c.x, a.x),
                        fmaf((v[u].y - mu) * rstd, 1.f + c.y, a.y),
                        fmaf((v[u].z - mu) * rstd, 1.f + c.z, a.z),
                        fmaf((v[u].w - mu) * rstd, 1.f + c.w, a.w)};
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) {
      const float4* wr = reinterpret_cast<const float4*>(f.W + (int64_t)(4 * i + j4) * P);
#pragma unroll
      for (int c4 = 0; c4 < P / 4; ++c4) {
        const float4 w = __ldg(wr + c4);
        acc[4 * c4] = fmaf(y[j4], w.x, acc[4 * c4]);
        acc[4 * c4 + 1] = fmaf(y[j4], w.y, acc[4 * c4 + 1]);
        acc[4 * c4 + 2] = fmaf(y[j4], w.z, acc[4 * c4 + 2]);
        acc[4 * c4 + 3] = fmaf(y[j4], w.w, acc[4 * c4 + 3]);
      }
    }
  }
  // fixed-order butterfly over the warp, then lane j scatters output j
#pragma unroll
  for (int j = 0; j < P; ++j) {
#pragma unroll
    for (int o = 16; o; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
  }
  float mine = 0.f;
#pragma unroll
  for (int j = 0; j < P; ++j)
    if ((j & 31) == lane) mine = acc[j];
  for (int j = lane; j < P; j += 32) {
    float out = j < 32 ? mine : 0.f;
    if (j >= 32) {  // P > 32: the second half (lane j - 32 already holds acc[j])
#pragma unroll
      for (int jj = 32; jj < P; ++jj)
        if (jj == j) out = acc[jj];
    }
    f.eps[(int64_t)b * f.n_latent + patch_elem_index(f.g, l, j)] = out + (f.bias ? f.bias[j] : 0.f);
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
  pdl_wait_and_release();
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

// Whole-sequence attention for short sequences (L <= AS_MAXL): the head's
// K and V live in smem for the whole CTA, CTA = 16 queries (4 warps x 4), so
// a (lane, head) pair spreads over L/16 CTAs. Lane j scores keys j + 32m,
// the probabilities go through a per-warp smem row, lane owns dims lane+32u.
constexpr int AS_Q = 16, AS_WARPS = 4, AS_MAXL = 512, AS_MAXM = AS_MAXL / 32;

static size_t attn_small_smem(int L, int dh) {
  return ((size_t)L * (dh + 1) + (size_t)L * dh + AS_Q * dh + AS_WARPS * L) * sizeof(float);
}

static __global__ void __launch_bounds__(AS_WARPS * 32)
    attn_small_kernel(const __grid_constant__ AttnArgs p) {
  extern __shared__ float as_s[];
  pdl_wait_and_release();
  const int dh = p.dh, ldk = dh + 1, L = p.L;
  float* Ks = as_s;                 // [L][dh+1]
  float* Vs = Ks + L * ldk;         // [L][dh]
  float* Qs = Vs + L * dh;          // [AS_Q][dh]
  float* Ps = Qs + AS_Q * dh;       // [AS_WARPS][L]
  const int head = blockIdx.y, b = blockIdx.z, q0 = blockIdx.x * AS_Q;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (int64_t)b * L;
  const int ld = 3 * p.D;
  const int dh4 = dh >> 2;  // dh % 4 == 0 (spec heads: 32/64/72/64)
  for (int idx = threadIdx.x; idx < L * dh4; idx += blockDim.x) {
    const int j = idx / dh4, d = (idx % dh4) * 4;
    const float* src = p.qkv + (row0 + j) * ld + head * dh + d;
    const float4 kv = *reinterpret_cast<const float4*>(src + p.D);
    const float4 vv = *reinterpret_cast<const float4*>(src + 2 * p.D);
    float* kd = Ks + j * ldk + d;
    kd[0] = kv.x; kd[1] = kv.y; kd[2] = kv.z; kd[3] = kv.w;
    *reinterpret_cast<float4*>(Vs + j * dh + d) = vv;
  }
  for (int idx = threadIdx.x; idx < AS_Q * dh; idx += blockDim.x) {
    const int r = idx / dh, d = idx % dh, q = q0 + r;
    Qs[idx] = q < L ? p.qkv[(row0 + q) * ld + head * dh + d] * p.scale : 0.f;
  }
  __syncthreads();
  const int nm = (L + 31) / 32;
  const int nU = (dh + 31) / 32;
  LnModArgs st{};
  st.out_f32 = p.out_f32;
  st.out_bf16 = p.out_bf16;
  st.out_hi = p.out_hi;
  st.out_lo = p.out_lo;
  float* prow = Ps + warp * L;
  for (int r = 0; r < AS_Q / AS_WARPS; ++r) {
    const int qr = warp * (AS_Q / AS_WARPS) + r, q = q0 + qr;
    if (q >= L) break;
    const float* qv = Qs + qr * dh;
    float s[AS_MAXM];
#pragma unroll
    for (int m = 0; m < AS_MAXM; ++m) s[m] = 0.f;
    for (int d = 0; d < dh; ++d) {
      const float x = qv[d];
#pragma unroll
      for (int m = 0; m < AS_MAXM; ++m)
        if (m < nm) s[m] = fmaf(x, Ks[(lane + 32 * m) * ldk + d], s[m]);
    }
    float mx = -INFINITY;
#pragma unroll
    for (int m = 0; m < AS_MAXM; ++m)
      if (m < nm && lane + 32 * m < L) mx = fmaxf(mx, s[m]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
#pragma unroll
    for (int m = 0; m < AS_MAXM; ++m) {
      if (m < nm) {
        const int j = lane + 32 * m;
        const float e = j < L ? expf(s[m] - mx) : 0.f;
        if (j < L) prow[j] = e;
        sum += e;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    __syncwarp();
    float o_acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < L; ++j) {
      const float pj = prow[j];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int d = lane + 32 * u;
        if (u < nU && d < dh) o_acc[u] = fmaf(pj, Vs[j * dh + d], o_acc[u]);
      }
    }
    const float inv = 1.f / sum;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int d = lane + 32 * u;
      if (u < nU && d < dh) store_act(st, (row0 + q) * p.D + head * dh + d, o_acc[u] * inv);
    }
    __syncwarp();
  }
}

}  // namespace ps
