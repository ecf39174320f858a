// Flash attention on tensor cores for the bf16 predictor path.
//
// softmax(Q K^T / sqrt(dh)) V per (lane b, head), any sequence length L,
// head_dim dh <= 128 with dh % 8 == 0 (DiT-XL/2: 72, CogVideoX-shaped: 64).
// CTA = 4 warps x 16 queries; key blocks of 64 staged in smem as bf16
// (K row-major, V transposed so both MMA B fragments are 32-bit loads);
// S = Q K^T and O += P V on bf16 MMAs (m16n8k16, fp32 accumulate) with the
// FA2 register trick (the S accumulator fragment is re-packed in place as
// the P operand); online softmax in fp32 with exp2. QK^T runs over dh padded
// to a multiple of 16 with zeros.
//
// qkv row m = [q(D) | k(D) | v(D)] fp32 from the QKV GEMM; the output row is
// written in the proj GEMM's operand format (bf16).
#pragma once

#include "dit_kernels.cuh"

namespace ps {

constexpr int FA_WARPS = 4, FA_QW = 16, FA_KB = 64, FA_MAXDH = 128;

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void mma_bf16_16816(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int DHP>  // dh padded to a multiple of 16 (K of QK^T)
__global__ void __launch_bounds__(FA_WARPS * 32) attn_mma_kernel(const __grid_constant__ AttnArgs p) {
  constexpr int KST = DHP + 8;        // K smem row stride (bf16), breaks bank conflicts
  constexpr int VST = FA_KB + 8;      // V^T smem row stride
  constexpr int NKT = DHP / 16;       // k-steps of QK^T
  constexpr int NOT = DHP / 8;        // max n-tiles of O (dh/8 used)
  __shared__ __align__(16) __nv_bfloat16 Ks[FA_KB * KST];
  __shared__ __align__(16) __nv_bfloat16 Vt[DHP * VST];

  const int dh = p.dh, L = p.L, ld = 3 * p.D;
  const int head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t row0 = (int64_t)b * L;
  const int q0 = blockIdx.x * (FA_WARPS * FA_QW) + warp * FA_QW;
  const float qscale = p.scale * 1.4426950408889634f;  // fold log2(e): softmax via exp2

  // Q fragments (A operand), scaled, zero beyond L / dh
  uint32_t qa[NKT][4];
  {
    const int r0 = q0 + gid, r1 = q0 + gid + 8;
#pragma unroll
    for (int ks = 0; ks < NKT; ++ks) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // h: column half (k0 or k0+8)
        const int d = ks * 16 + h * 8 + tig * 2;
        float a0 = 0.f, a1 = 0.f, c0 = 0.f, c1 = 0.f;
        if (d < dh) {
          if (r0 < L) {
            const float* src = p.qkv + (row0 + r0) * ld + head * dh + d;
            a0 = src[0] * qscale;
            a1 = src[1] * qscale;
          }
          if (r1 < L) {
            const float* src = p.qkv + (row0 + r1) * ld + head * dh + d;
            c0 = src[0] * qscale;
            c1 = src[1] * qscale;
          }
        }
        qa[ks][2 * h] = pack_bf16(a0, a1);
        qa[ks][2 * h + 1] = pack_bf16(c0, c1);
      }
    }
  }
  float o[NOT][4];
#pragma unroll
  for (int t = 0; t < NOT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int k0 = 0; k0 < L; k0 += FA_KB) {
    __syncthreads();
    // stage K (row-major) and V^T for keys k0..k0+63 as bf16, zero padded
    for (int idx = threadIdx.x; idx < FA_KB * (DHP / 2); idx += blockDim.x) {
      const int j = idx / (DHP / 2), d = (idx % (DHP / 2)) * 2, kk = k0 + j;
      float k_a = 0.f, k_b = 0.f, v_a = 0.f, v_b = 0.f;
      if (kk < L && d < dh) {
        const float* src = p.qkv + (row0 + kk) * ld + head * dh + d;
        const float2 kv = *reinterpret_cast<const float2*>(src + p.D);
        const float2 vv = *reinterpret_cast<const float2*>(src + 2 * p.D);
        k_a = kv.x; k_b = kv.y; v_a = vv.x; v_b = vv.y;
      }
      *reinterpret_cast<uint32_t*>(&Ks[j * KST + d]) = pack_bf16(k_a, k_b);
      Vt[d * VST + j] = __float2bfloat16_rn(v_a);
      Vt[(d + 1) * VST + j] = __float2bfloat16_rn(v_b);
    }
    __syncthreads();
    // S = Q K^T : 8 n-tiles of 8 keys
    float s[FA_KB / 8][4];
#pragma unroll
    for (int nt = 0; nt < FA_KB / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < NKT; ++ks) {
        const __nv_bfloat16* kp = Ks + (nt * 8 + gid) * KST + ks * 16 + tig * 2;
        uint32_t bfrag[2] = {*reinterpret_cast<const uint32_t*>(kp),
                             *reinterpret_cast<const uint32_t*>(kp + 8)};
        mma_bf16_16816(s[nt], qa[ks], bfrag);
      }
    }
    // mask keys beyond L, online softmax (rows gid and gid+8)
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nt = 0; nt < FA_KB / 8; ++nt) {
      const int kk = k0 + nt * 8 + tig * 2;
      if (kk >= L) { s[nt][0] = -INFINITY; s[nt][2] = -INFINITY; }
      if (kk + 1 >= L) { s[nt][1] = -INFINITY; s[nt][3] = -INFINITY; }
      mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
    }
#pragma unroll
    for (int o_ = 1; o_ <= 2; o_ <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o_));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o_));
    }
    const float c0 = exp2f(m0 - mx0), c1 = exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pa[FA_KB / 16][4];
#pragma unroll
    for (int nt = 0; nt < FA_KB / 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - mx0), p1 = exp2f(s[nt][1] - mx0);
      const float p2 = exp2f(s[nt][2] - mx1), p3 = exp2f(s[nt][3] - mx1);
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      const int kt = nt >> 1, hh = nt & 1;
      pa[kt][2 * hh] = pack_bf16(p0, p1);
      pa[kt][2 * hh + 1] = pack_bf16(p2, p3);
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int t = 0; t < NOT; ++t) {
      o[t][0] *= c0; o[t][1] *= c0;
      o[t][2] *= c1; o[t][3] *= c1;
    }
    // O += P V : k-steps of 16 keys, n-tiles of 8 dims
#pragma unroll
    for (int kt = 0; kt < FA_KB / 16; ++kt) {
#pragma unroll
      for (int t = 0; t < NOT; ++t) {
        if (t * 8 < dh) {
          const __nv_bfloat16* vp = Vt + (t * 8 + gid) * VST + kt * 16 + tig * 2;
          uint32_t bfrag[2] = {*reinterpret_cast<const uint32_t*>(vp),
                               *reinterpret_cast<const uint32_t*>(vp + 8)};
          mma_bf16_16816(o[t], pa[kt], bfrag);
        }
      }
    }
  }
  // finalize: row sums across the 4 threads of a row group
#pragma unroll
  for (int o_ = 1; o_ <= 2; o_ <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o_);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o_);
  }
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  LnModArgs st{};
  st.out_f32 = p.out_f32;
  st.out_bf16 = p.out_bf16;
  st.out_hi = p.out_hi;
  st.out_lo = p.out_lo;
  const int r0 = q0 + gid, r1 = q0 + gid + 8;
#pragma unroll
  for (int t = 0; t < NOT; ++t) {
    const int d = t * 8 + tig * 2;
    if (d < dh) {
      if (r0 < L) {
        const int64_t idx = (row0 + r0) * p.D + head * dh + d;
        store_act(st, idx, o[t][0] * i0);
        store_act(st, idx + 1, o[t][1] * i0);
      }
      if (r1 < L) {
        const int64_t idx = (row0 + r1) * p.D + head * dh + d;
        store_act(st, idx, o[t][2] * i1);
        store_act(st, idx + 1, o[t][3] * i1);
      }
    }
  }
}

// dispatch on padded head dim; returns false if unsupported
static inline bool launch_attn_mma(const AttnArgs& a, int B, cudaStream_t st) {
  const int dhp = (a.dh + 15) / 16 * 16;
  dim3 grid((a.L + FA_WARPS * FA_QW - 1) / (FA_WARPS * FA_QW), a.H, B);
  switch (dhp) {
    case 32: attn_mma_kernel<32><<<grid, FA_WARPS * 32, 0, st>>>(a); return true;
    case 48: attn_mma_kernel<48><<<grid, FA_WARPS * 32, 0, st>>>(a); return true;
    case 64: attn_mma_kernel<64><<<grid, FA_WARPS * 32, 0, st>>>(a); return true;
    case 80: attn_mma_kernel<80><<<grid, FA_WARPS * 32, 0, st>>>(a); return true;
    case 96: attn_mma_kernel<96><<<grid, FA_WARPS * 32, 0, st>>>(a); return true;
    case 128: attn_mma_kernel<128><<<grid, FA_WARPS * 32, 0, st>>>(a); return true;
    default: return false;
  }
}

}  // namespace ps

// ---------------------------------------------------------------------------
// fp32-accurate variant for the fp32 predictor path: the same flash
// structure on tf32 MMAs (m16n8k8) with the 3-pass split x = hi + lo
// (hi*hi + hi*lo + lo*hi) for both QK^T and PV. The S accumulator fragment
// holds columns {2t, 2t+1} while the tf32 A fragment wants {t, t+4}; instead
// of shuffling, the 8 keys of each group are consumed in the permuted order
// sigma(t) = 2t, sigma(t+4) = 2t+1 on both P and V, which leaves P.V unchanged.
namespace ps {

__device__ __forceinline__ uint32_t tf32_bits(float v) { return __float_as_uint(v) & 0xFFFFE000u; }

__device__ __forceinline__ void split_tf32(float v, uint32_t& hi, uint32_t& lo) {
  hi = tf32_bits(v);
  lo = __float_as_uint(v - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32_1688(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ void mma3(float* c, const uint32_t* ah, const uint32_t* al,
                                     const uint32_t* bh, const uint32_t* bl) {
  mma_tf32_1688(c, al, bh);
  mma_tf32_1688(c, ah, bl);
  mma_tf32_1688(c, ah, bh);
}

template <int DHP>  // dh padded to a multiple of 8
__global__ void __launch_bounds__(FA_WARPS * 32) attn_tf32x3_kernel(const __grid_constant__ AttnArgs p) {
  constexpr int KST = DHP + 4;   // K smem row stride (floats): conflict-free frag loads
  constexpr int VST = FA_KB + 8; // V^T row stride (floats)
  constexpr int NKT = DHP / 8;
  constexpr int NOT = DHP / 8;
  __shared__ __align__(16) float Ks[FA_KB * KST];
  __shared__ __align__(16) float Vt[DHP * VST];

  const int dh = p.dh, L = p.L, ld = 3 * p.D;
  const int head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t row0 = (int64_t)b * L;
  const int q0 = blockIdx.x * (FA_WARPS * FA_QW) + warp * FA_QW;

  uint32_t qh[NKT][4], ql[NKT][4];
  {
    const int r0 = q0 + gid, r1 = q0 + gid + 8;
#pragma unroll
    for (int ks = 0; ks < NKT; ++ks) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // a0/a1: col tig, a2/a3: col tig+4
        const int d = ks * 8 + tig + 4 * h;
        float v0 = 0.f, v1 = 0.f;
        if (d < dh) {
          if (r0 < L) v0 = p.qkv[(row0 + r0) * ld + head * dh + d] * p.scale;
          if (r1 < L) v1 = p.qkv[(row0 + r1) * ld + head * dh + d] * p.scale;
        }
        split_tf32(v0, qh[ks][2 * h], ql[ks][2 * h]);
        split_tf32(v1, qh[ks][2 * h + 1], ql[ks][2 * h + 1]);
      }
    }
  }
  float o[NOT][4];
#pragma unroll
  for (int t = 0; t < NOT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int k0 = 0; k0 < L; k0 += FA_KB) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < FA_KB * (DHP / 4); idx += blockDim.x) {
      const int j = idx / (DHP / 4), d = (idx % (DHP / 4)) * 4, kk = k0 + j;
      float4 kv = make_float4(0.f, 0.f, 0.f, 0.f), vv = kv;
      if (kk < L && d < dh) {
        const float* src = p.qkv + (row0 + kk) * ld + head * dh + d;
        kv = *reinterpret_cast<const float4*>(src + p.D);
        vv = *reinterpret_cast<const float4*>(src + 2 * p.D);
      }
      *reinterpret_cast<float4*>(&Ks[j * KST + d]) = kv;
      Vt[(d + 0) * VST + j] = vv.x;
      Vt[(d + 1) * VST + j] = vv.y;
      Vt[(d + 2) * VST + j] = vv.z;
      Vt[(d + 3) * VST + j] = vv.w;
    }
    __syncthreads();
    float s[FA_KB / 8][4];
#pragma unroll
    for (int nt = 0; nt < FA_KB / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < NKT; ++ks) {
        const float* kp = Ks + (nt * 8 + gid) * KST + ks * 8 + tig;
        uint32_t bh[2], bl[2];
        split_tf32(kp[0], bh[0], bl[0]);
        split_tf32(kp[4], bh[1], bl[1]);
        mma3(s[nt], qh[ks], ql[ks], bh, bl);
      }
    }
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nt = 0; nt < FA_KB / 8; ++nt) {
      const int kk = k0 + nt * 8 + tig * 2;
      if (kk >= L) { s[nt][0] = -INFINITY; s[nt][2] = -INFINITY; }
      if (kk + 1 >= L) { s[nt][1] = -INFINITY; s[nt][3] = -INFINITY; }
      mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
    }
#pragma unroll
    for (int o_ = 1; o_ <= 2; o_ <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o_));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o_));
    }
    const float c0 = expf(m0 - mx0), c1 = expf(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int t = 0; t < NOT; ++t) {
      o[t][0] *= c0; o[t][1] *= c0;
      o[t][2] *= c1; o[t][3] *= c1;
    }
#pragma unroll
    for (int nt = 0; nt < FA_KB / 8; ++nt) {
      const float p0 = expf(s[nt][0] - mx0), p1 = expf(s[nt][1] - mx0);
      const float p2 = expf(s[nt][2] - mx1), p3 = expf(s[nt][3] - mx1);
      rs0 += p0 + p1;
      rs1 += p2 + p3;
      // A fragment in the permuted key order: a0 = P[g][2t], a1 = P[g+8][2t],
      // a2 = P[g][2t+1], a3 = P[g+8][2t+1]
      uint32_t ah[4], al[4];
      split_tf32(p0, ah[0], al[0]);
      split_tf32(p2, ah[1], al[1]);
      split_tf32(p1, ah[2], al[2]);
      split_tf32(p3, ah[3], al[3]);
#pragma unroll
      for (int t = 0; t < NOT; ++t) {
        if (t * 8 < dh) {
          const float2 v2 = *reinterpret_cast<const float2*>(Vt + (t * 8 + gid) * VST + nt * 8 + tig * 2);
          uint32_t bh[2], bl[2];
          split_tf32(v2.x, bh[0], bl[0]);  // key 2t   (A column t)
          split_tf32(v2.y, bh[1], bl[1]);  // key 2t+1 (A column t+4)
          mma3(o[t], ah, al, bh, bl);
        }
      }
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
  }
#pragma unroll
  for (int o_ = 1; o_ <= 2; o_ <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o_);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o_);
  }
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  LnModArgs st{};
  st.out_f32 = p.out_f32;
  st.out_bf16 = p.out_bf16;
  st.out_hi = p.out_hi;
  st.out_lo = p.out_lo;
  const int r0 = q0 + gid, r1 = q0 + gid + 8;
#pragma unroll
  for (int t = 0; t < NOT; ++t) {
    const int d = t * 8 + tig * 2;
    if (d < dh) {
      if (r0 < L) {
        const int64_t idx = (row0 + r0) * p.D + head * dh + d;
        store_act(st, idx, o[t][0] * i0);
        store_act(st, idx + 1, o[t][1] * i0);
      }
      if (r1 < L) {
        const int64_t idx = (row0 + r1) * p.D + head * dh + d;
        store_act(st, idx, o[t][2] * i1);
        store_act(st, idx + 1, o[t][3] * i1);
      }
    }
  }
}

static inline bool launch_attn_tf32x3(const AttnArgs& a, int B, cudaStream_t st) {
  const int dhp = (a.dh + 7) / 8 * 8;
  dim3 grid((a.L + FA_WARPS * FA_QW - 1) / (FA_WARPS * FA_QW), a.H, B);
  switch (dhp) {
    case 32: attn_tf32x3_kernel<32><<<grid, FA_WARPS * 32, 0, st>>>(a); return true;
    case 64: attn_tf32x3_kernel<64><<<grid, FA_WARPS * 32, 0, st>>>(a); return true;
    case 72: attn_tf32x3_kernel<72><<<grid, FA_WARPS * 32, 0, st>>>(a); return true;
    default: return false;
  }
}

}  // namespace ps
