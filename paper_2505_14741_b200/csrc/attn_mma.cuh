// Flash attention on tensor cores (both predictor precisions).
//
// softmax(Q K^T / sqrt(dh)) V per (lane b, head), any sequence length L,
// head_dim dh % 8 == 0 (DiT-S/2 64, DiT-XL/2 72, CogVideoX-shaped 64).
// CTA = NW warps x 16 queries. Key blocks of 64 rows of K and V are staged
// fp32 into a 2-stage smem ring with cp.async (16 B, zero-fill past L), so
// the next block streams in while the current one is on the tensor cores.
// S = Q K^T and O += P V run on mma.sync with fp32 accumulation; online
// softmax in fp32; the S accumulator fragment is reused in registers as the
// P operand (FA2). Two arithmetic modes:
//   AM_BF16   m16n8k16 bf16 (bf16 path; exp2 with log2e folded into Q)
//   AM_TF32X3 m16n8k8 tf32 with the 3-pass split x = hi + lo for both MMAs
//             (fp32 path, error ~1e-6); the S fragment holds columns
//             {2t, 2t+1} and the tf32 A fragment wants {t, t+4}, so each
//             8-key group is consumed in the permuted order s(t) = 2t,
//             s(t+4) = 2t+1 on P and V alike (P.V unchanged, no shuffles).
// qkv row m = [q(D) | k(D) | v(D)] fp32 from the QKV GEMM; the output row is
// written in the proj GEMM's operand format.
#pragma once

#include <cstdlib>

#include "dit_kernels.cuh"

namespace ps {

enum { AM_BF16 = 0, AM_TF32X3 = 1 };
constexpr int FA_QW = 16, FA_KB = 64;

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

__device__ __forceinline__ void mma_tf32_1688(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ void split_tf32(float v, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(v) & 0xFFFFE000u;
  lo = __float_as_uint(v - __uint_as_float(hi));
}

// small terms first: lo*hi + hi*lo + hi*hi
__device__ __forceinline__ void mma3(float* c, const uint32_t* ah, const uint32_t* al,
                                     const uint32_t* bh, const uint32_t* bl) {
  mma_tf32_1688(c, al, bh);
  mma_tf32_1688(c, ah, bl);
  mma_tf32_1688(c, ah, bh);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int DHP>
struct FaCfg {
  static constexpr int ST = DHP + 4;                 // smem row stride (floats), 16 B multiple
  static constexpr int STAGE = 2 * FA_KB * ST;       // K block + V block (floats)
  static constexpr size_t SMEM = 2 * STAGE * sizeof(float);
};

template <int MODE, int DHP, int NW>
__global__ void __launch_bounds__(NW * 32) attn_tc_kernel(const __grid_constant__ AttnArgs p) {
  using C = FaCfg<DHP>;
  constexpr int ST = C::ST;
  constexpr int NOT = DHP / 8;  // output n-tiles (only t*8 < dh used)
  extern __shared__ __align__(16) float fa_smem[];
  pdl_wait_and_release();

  const int dh = p.dh, L = p.L, ld = 3 * p.D;
  const int head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t row0 = (int64_t)b * L;
  const int q0 = blockIdx.x * (NW * FA_QW) + warp * FA_QW;
  const int nkb = (L + FA_KB - 1) / FA_KB;
  const int dh4 = dh >> 2;

  // zero the pad columns [dh, DHP) of both stages once (cp.async never writes them)
  if (DHP > dh) {
    for (int idx = threadIdx.x; idx < 2 * 2 * FA_KB; idx += NW * 32)
      for (int d = dh; d < DHP; ++d) fa_smem[idx * ST + d] = 0.f;
  }
  auto stage_load = [&](int kb, int stg) {
    float* Kd = fa_smem + stg * C::STAGE;
    float* Vd = Kd + FA_KB * ST;
    for (int idx = threadIdx.x; idx < FA_KB * dh4; idx += NW * 32) {
      const int j = idx / dh4, c4 = (idx % dh4) * 4, kk = kb * FA_KB + j;
      const int ok = kk < L ? 16 : 0;
      const float* src = p.qkv + (row0 + (kk < L ? kk : 0)) * ld + head * dh + c4;
      cp_async16(Kd + j * ST + c4, src + p.D, ok);
      cp_async16(Vd + j * ST + c4, src + 2 * p.D, ok);
    }
    cp_async_commit();
  };
  stage_load(0, 0);

  // Q fragments, pre-scaled (bf16: log2e folded in for exp2 softmax)
  const float qscale = MODE == AM_BF16 ? p.scale * 1.4426950408889634f : p.scale;
  const int r0 = q0 + gid, r1 = q0 + gid + 8;
  auto qval = [&](int r, int d) -> float {
    return (r < L && d < dh) ? p.qkv[(row0 + r) * ld + head * dh + d] * qscale : 0.f;
  };
  constexpr int NKS = MODE == AM_BF16 ? DHP / 16 : DHP / 8;  // k-steps of QK^T
  uint32_t qh[NKS][4], ql[MODE == AM_BF16 ? 1 : NKS][4];
#pragma unroll
  for (int ks = 0; ks < NKS; ++ks) {
    if constexpr (MODE == AM_BF16) {
      const int d = ks * 16 + tig * 2;
      qh[ks][0] = pack_bf16(qval(r0, d), qval(r0, d + 1));
      qh[ks][1] = pack_bf16(qval(r1, d), qval(r1, d + 1));
      qh[ks][2] = pack_bf16(qval(r0, d + 8), qval(r0, d + 9));
      qh[ks][3] = pack_bf16(qval(r1, d + 8), qval(r1, d + 9));
    } else {
      const int d = ks * 8 + tig;
      split_tf32(qval(r0, d), qh[ks][0], ql[ks][0]);
      split_tf32(qval(r1, d), qh[ks][1], ql[ks][1]);
      split_tf32(qval(r0, d + 4), qh[ks][2], ql[ks][2]);
      split_tf32(qval(r1, d + 4), qh[ks][3], ql[ks][3]);
    }
  }
  float o[NOT][4];
#pragma unroll
  for (int t = 0; t < NOT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int kb = 0; kb < nkb; ++kb) {
    if (kb + 1 < nkb) {
      stage_load(kb + 1, (kb + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* Ks = fa_smem + (kb & 1) * C::STAGE;
    const float* Vs = Ks + FA_KB * ST;
    const int k0 = kb * FA_KB;

    float s[FA_KB / 8][4];
#pragma unroll
    for (int nt = 0; nt < FA_KB / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
      const float* kr = Ks + (nt * 8 + gid) * ST;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        if constexpr (MODE == AM_BF16) {
          const float2 a = *reinterpret_cast<const float2*>(kr + ks * 16 + tig * 2);
          const float2 c = *reinterpret_cast<const float2*>(kr + ks * 16 + 8 + tig * 2);
          uint32_t bf[2] = {pack_bf16(a.x, a.y), pack_bf16(c.x, c.y)};
          mma_bf16_16816(s[nt], qh[ks], bf);
        } else {
          uint32_t bh[2], bl[2];
          split_tf32(kr[ks * 8 + tig], bh[0], bl[0]);
          split_tf32(kr[ks * 8 + tig + 4], bh[1], bl[1]);
          mma3(s[nt], qh[ks], ql[ks], bh, bl);
        }
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
    const float c0 = MODE == AM_BF16 ? exp2f(m0 - mx0) : expf(m0 - mx0);
    const float c1 = MODE == AM_BF16 ? exp2f(m1 - mx1) : expf(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
#pragma unroll
    for (int t = 0; t < NOT; ++t) {
      o[t][0] *= c0; o[t][1] *= c0;
      o[t][2] *= c1; o[t][3] *= c1;
    }
    float rs0 = 0.f, rs1 = 0.f;
    if constexpr (MODE == AM_BF16) {
      uint32_t pa[FA_KB / 16][4];
#pragma unroll
      for (int nt = 0; nt < FA_KB / 8; ++nt) {
        const float p0 = exp2f(s[nt][0] - mx0), p1 = exp2f(s[nt][1] - mx0);
        const float p2 = exp2f(s[nt][2] - mx1), p3 = exp2f(s[nt][3] - mx1);
        rs0 += p0 + p1;
        rs1 += p2 + p3;
        pa[nt >> 1][2 * (nt & 1)] = pack_bf16(p0, p1);
        pa[nt >> 1][2 * (nt & 1) + 1] = pack_bf16(p2, p3);
      }
#pragma unroll
      for (int kt = 0; kt < FA_KB / 16; ++kt) {
        const float* v0 = Vs + (kt * 16 + tig * 2) * ST;
#pragma unroll
        for (int t = 0; t < NOT; ++t) {
          if (t * 8 < dh) {
            const int d = t * 8 + gid;
            uint32_t bf[2] = {pack_bf16(v0[d], v0[ST + d]),
                              pack_bf16(v0[8 * ST + d], v0[9 * ST + d])};
            mma_bf16_16816(o[t], pa[kt], bf);
          }
        }
      }
    } else {
#pragma unroll
      for (int nt = 0; nt < FA_KB / 8; ++nt) {
        const float p0 = expf(s[nt][0] - mx0), p1 = expf(s[nt][1] - mx0);
        const float p2 = expf(s[nt][2] - mx1), p3 = expf(s[nt][3] - mx1);
        rs0 += p0 + p1;
        rs1 += p2 + p3;
        uint32_t ah[4], al[4];  // permuted order: a0 = P[g][2t], a2 = P[g][2t+1]
        split_tf32(p0, ah[0], al[0]);
        split_tf32(p2, ah[1], al[1]);
        split_tf32(p1, ah[2], al[2]);
        split_tf32(p3, ah[3], al[3]);
        const float* v0 = Vs + (nt * 8 + tig * 2) * ST;
#pragma unroll
        for (int t = 0; t < NOT; ++t) {
          if (t * 8 < dh) {
            const int d = t * 8 + gid;
            uint32_t bh[2], bl[2];
            split_tf32(v0[d], bh[0], bl[0]);       // key 2t   (A column t)
            split_tf32(v0[ST + d], bh[1], bl[1]);  // key 2t+1 (A column t+4)
            mma3(o[t], ah, al, bh, bl);
          }
        }
      }
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
    __syncthreads();  // the stage is overwritten by the next prefetch
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

// ---------------------------------------------------------------------------
// Key-split variant for short sequences (the DiT-S/2 and DiT-XL/2 shapes,
// L = 256): a CTA owns ONE 16-query tile and its KW warps split the keys
// (warp w takes 32-key blocks w, w+KW, ...), each with a private 2-stage
// cp.async ring, then merge their (max, sum, O) partials through smem in warp
// order (deterministic). 4x more warps in flight than one warp per query
// tile, which is what a latency-bound L = 256 attention needs.
constexpr int KS_KB = 32;
constexpr int KS_KW_DEFAULT = 8;  // measured: 8 warps x one 32-key block beat 4 x two at L=256

template <int DHP>
struct KsCfg {
  static constexpr int ST = DHP + 4;
  static constexpr int WSTAGE = 2 * KS_KB * ST;  // K + V floats per stage per warp
  // stages per warp: 2 (double-buffered loop over key blocks), or 1 when the
  // 8-warp variant covers the whole sequence with one block per warp
  static constexpr int nst(int kw) { return kw == 8 ? 1 : 2; }
  static size_t smem(int kw) { return (size_t)kw * nst(kw) * WSTAGE * sizeof(float); }
};

template <int MODE, int DHP, int KW>
__global__ void __launch_bounds__(KW * 32) attn_ks_kernel(const __grid_constant__ AttnArgs p) {
  using C = KsCfg<DHP>;
  constexpr int ST = C::ST;
  constexpr int NOT = DHP / 8;
  extern __shared__ __align__(16) float ks_smem[];
  pdl_wait_and_release();

  const int dh = p.dh, L = p.L, ld = 3 * p.D;
  const int head = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t row0 = (int64_t)b * L;
  const int q0 = blockIdx.x * FA_QW;
  const int nkb = (L + KS_KB - 1) / KS_KB;
  const int dh4 = dh >> 2;
  constexpr int NST = C::nst(KW);
  float* wbuf = ks_smem + (size_t)warp * NST * C::WSTAGE;

  if (DHP > dh)  // zero the pad columns of this warp's stages once
    for (int r = lane; r < NST * 2 * KS_KB; r += 32)
      for (int d = dh; d < DHP; ++d) wbuf[r * ST + d] = 0.f;
  auto stage_load = [&](int kb, int stg) {
    float* Kd = wbuf + stg * C::WSTAGE;
    float* Vd = Kd + KS_KB * ST;
    for (int idx = lane; idx < KS_KB * dh4; idx += 32) {
      const int j = idx / dh4, c4 = (idx % dh4) * 4, kk = kb * KS_KB + j;
      const int ok = kk < L ? 16 : 0;
      const float* src = p.qkv + (row0 + (kk < L ? kk : 0)) * ld + head * dh + c4;
      cp_async16(Kd + j * ST + c4, src + p.D, ok);
      cp_async16(Vd + j * ST + c4, src + 2 * p.D, ok);
    }
    cp_async_commit();
  };
  if (warp < nkb) stage_load(warp, 0);

  const float qscale = MODE == AM_BF16 ? p.scale * 1.4426950408889634f : p.scale;
  const int r0 = q0 + gid, r1 = q0 + gid + 8;
  auto qval = [&](int r, int d) -> float {
    return (r < L && d < dh) ? p.qkv[(row0 + r) * ld + head * dh + d] * qscale : 0.f;
  };
  constexpr int NKS = MODE == AM_BF16 ? DHP / 16 : DHP / 8;
  uint32_t qh[NKS][4], ql[MODE == AM_BF16 ? 1 : NKS][4];
#pragma unroll
  for (int ks = 0; ks < NKS; ++ks) {
    if constexpr (MODE == AM_BF16) {
      const int d = ks * 16 + tig * 2;
      qh[ks][0] = pack_bf16(qval(r0, d), qval(r0, d + 1));
      qh[ks][1] = pack_bf16(qval(r1, d), qval(r1, d + 1));
      qh[ks][2] = pack_bf16(qval(r0, d + 8), qval(r0, d + 9));
      qh[ks][3] = pack_bf16(qval(r1, d + 8), qval(r1, d + 9));
    } else {
      const int d = ks * 8 + tig;
      split_tf32(qval(r0, d), qh[ks][0], ql[ks][0]);
      split_tf32(qval(r1, d), qh[ks][1], ql[ks][1]);
      split_tf32(qval(r0, d + 4), qh[ks][2], ql[ks][2]);
      split_tf32(qval(r1, d + 4), qh[ks][3], ql[ks][3]);
    }
  }
  float o[NOT][4];
#pragma unroll
  for (int t = 0; t < NOT; ++t) o[t][0] = o[t][1] = o[t][2] = o[t][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  int it = 0;
  for (int kb = warp; kb < nkb; kb += KW, ++it) {
    if (kb + KW < nkb) {
      stage_load(kb + KW, (it + 1) % NST);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const float* Ks = wbuf + (it % NST) * C::WSTAGE;
    const float* Vs = Ks + KS_KB * ST;
    const int k0 = kb * KS_KB;
    float s[KS_KB / 8][4];
#pragma unroll
    for (int nt = 0; nt < KS_KB / 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
      const float* kr = Ks + (nt * 8 + gid) * ST;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        if constexpr (MODE == AM_BF16) {
          const float2 a = *reinterpret_cast<const float2*>(kr + ks * 16 + tig * 2);
          const float2 c = *reinterpret_cast<const float2*>(kr + ks * 16 + 8 + tig * 2);
          uint32_t bf[2] = {pack_bf16(a.x, a.y), pack_bf16(c.x, c.y)};
          mma_bf16_16816(s[nt], qh[ks], bf);
        } else {
          uint32_t bh[2], bl[2];
          split_tf32(kr[ks * 8 + tig], bh[0], bl[0]);
          split_tf32(kr[ks * 8 + tig + 4], bh[1], bl[1]);
          mma3(s[nt], qh[ks], ql[ks], bh, bl);
        }
      }
    }
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nt = 0; nt < KS_KB / 8; ++nt) {
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
    const float c0 = MODE == AM_BF16 ? exp2f(m0 - mx0) : expf(m0 - mx0);
    const float c1 = MODE == AM_BF16 ? exp2f(m1 - mx1) : expf(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
#pragma unroll
    for (int t = 0; t < NOT; ++t) {
      o[t][0] *= c0; o[t][1] *= c0;
      o[t][2] *= c1; o[t][3] *= c1;
    }
    float rs0 = 0.f, rs1 = 0.f;
    if constexpr (MODE == AM_BF16) {
      uint32_t pa[KS_KB / 16][4];
#pragma unroll
      for (int nt = 0; nt < KS_KB / 8; ++nt) {
        const float p0 = exp2f(s[nt][0] - mx0), p1 = exp2f(s[nt][1] - mx0);
        const float p2 = exp2f(s[nt][2] - mx1), p3 = exp2f(s[nt][3] - mx1);
        rs0 += p0 + p1;
        rs1 += p2 + p3;
        pa[nt >> 1][2 * (nt & 1)] = pack_bf16(p0, p1);
        pa[nt >> 1][2 * (nt & 1) + 1] = pack_bf16(p2, p3);
      }
#pragma unroll
      for (int kt = 0; kt < KS_KB / 16; ++kt) {
        const float* v0 = Vs + (kt * 16 + tig * 2) * ST;
#pragma unroll
        for (int t = 0; t < NOT; ++t) {
          if (t * 8 < dh) {
            const int d = t * 8 + gid;
            uint32_t bf[2] = {pack_bf16(v0[d], v0[ST + d]),
                              pack_bf16(v0[8 * ST + d], v0[9 * ST + d])};
            mma_bf16_16816(o[t], pa[kt], bf);
          }
        }
      }
    } else {
#pragma unroll
      for (int nt = 0; nt < KS_KB / 8; ++nt) {
        const float p0 = expf(s[nt][0] - mx0), p1 = expf(s[nt][1] - mx0);
        const float p2 = expf(s[nt][2] - mx1), p3 = expf(s[nt][3] - mx1);
        rs0 += p0 + p1;
        rs1 += p2 + p3;
        uint32_t ah[4], al[4];
        split_tf32(p0, ah[0], al[0]);
        split_tf32(p2, ah[1], al[1]);
        split_tf32(p1, ah[2], al[2]);
        split_tf32(p3, ah[3], al[3]);
        const float* v0 = Vs + (nt * 8 + tig * 2) * ST;
#pragma unroll
        for (int t = 0; t < NOT; ++t) {
          if (t * 8 < dh) {
            const int d = t * 8 + gid;
            uint32_t bh[2], bl[2];
            split_tf32(v0[d], bh[0], bl[0]);
            split_tf32(v0[ST + d], bh[1], bl[1]);
            mma3(o[t], ah, al, bh, bl);
          }
        }
      }
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
    __syncwarp();  // this stage is refilled two blocks later
  }
#pragma unroll
  for (int o_ = 1; o_ <= 2; o_ <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, o_);
    l1 += __shfl_xor_sync(0xffffffffu, l1, o_);
  }
  // ---- merge the KW partials (warp order): smem reused after all warps finish
  __syncthreads();
  float* ms = ks_smem;                 // [KW][16]
  float* ls = ms + KW * FA_QW;         // [KW][16]
  float* os = ls + KW * FA_QW;         // [KW][16][DHP]
  if (tig == 0) {
    ms[warp * FA_QW + gid] = m0;
    ms[warp * FA_QW + gid + 8] = m1;
    ls[warp * FA_QW + gid] = l0;
    ls[warp * FA_QW + gid + 8] = l1;
  }
#pragma unroll
  for (int t = 0; t < NOT; ++t) {
    const int d = t * 8 + tig * 2;
    if (d < dh) {
      float* orow0 = os + ((size_t)warp * FA_QW + gid) * DHP + d;
      float* orow1 = os + ((size_t)warp * FA_QW + gid + 8) * DHP + d;
      orow0[0] = o[t][0];
      orow0[1] = o[t][1];
      orow1[0] = o[t][2];
      orow1[1] = o[t][3];
    }
  }
  __syncthreads();
  // per-row merge weights f_w = exp(m_w - M) and denominators, once per row
  // (not once per output element), same operations in the same order
  float* fs = os + (size_t)KW * FA_QW * DHP;  // [KW][16]
  float* dens = fs + KW * FA_QW;              // [16]
  if (threadIdx.x < FA_QW) {
    const int r = threadIdx.x;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < KW; ++w) M = fmaxf(M, ms[w * FA_QW + r]);
    float den = 0.f;
#pragma unroll
    for (int w = 0; w < KW; ++w) {
      const float mw = ms[w * FA_QW + r];
      const float f = mw == -INFINITY ? 0.f
                                      : (MODE == AM_BF16 ? exp2f(mw - M) : expf(mw - M));
      fs[w * FA_QW + r] = f;
      den = fmaf(ls[w * FA_QW + r], f, den);
    }
    dens[r] = den;
  }
  __syncthreads();
  LnModArgs st{};
  st.out_f32 = p.out_f32;
  st.out_bf16 = p.out_bf16;
  st.out_hi = p.out_hi;
  st.out_lo = p.out_lo;
  for (int idx = threadIdx.x; idx < FA_QW * dh; idx += KW * 32) {
    const int r = idx / dh, d = idx % dh, q = q0 + r;
    if (q >= L) continue;
    float num = 0.f;
#pragma unroll
    for (int w = 0; w < KW; ++w)
      num = fmaf(os[((size_t)w * FA_QW + r) * DHP + d], fs[w * FA_QW + r], num);
    store_act(st, (row0 + q) * p.D + head * dh + d, num / dens[r]);
  }
}

// warps per CTA of the key-split kernel (keys split KW ways). Tuned on B200
// (profiles/r1b_attn_probe.txt); PS_ATTN_KS_WARPS=4|8 overrides for probes.
static inline int ks_warps() {
  static int kw = [] {
    const char* e = getenv("PS_ATTN_KS_WARPS");
    return (e && atoi(e) == 8) ? 8 : (e && atoi(e) == 4 ? 4 : KS_KW_DEFAULT);
  }();
  return kw;
}

template <int MODE, int DHP, int KW>
static inline void launch_ks_w(const AttnArgs& a, int B, cudaStream_t st) {
  const size_t smem = KsCfg<DHP>::smem(KW);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_ks_kernel<MODE, DHP, KW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  dim3 grid((a.L + FA_QW - 1) / FA_QW, a.H, B);
  launch_pdl(attn_ks_kernel<MODE, DHP, KW>, grid, dim3(KW * 32), smem, st, a);
}

template <int MODE, int DHP>
static inline void launch_ks(const AttnArgs& a, int B, cudaStream_t st) {
  // the 8-warp variant is single-buffered: one 32-key block per warp
  if (ks_warps() == 8 && a.L <= 8 * KS_KB) launch_ks_w<MODE, DHP, 8>(a, B, st);
  else launch_ks_w<MODE, DHP, 4>(a, B, st);
}

constexpr int FA_NW = 2;  // 32 queries per CTA: more CTAs for short sequences

template <int MODE, int DHP>
static inline void launch_fa(const AttnArgs& a, int B, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_tc_kernel<MODE, DHP, FA_NW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FaCfg<DHP>::SMEM);
    attr = true;
  }
  dim3 grid((a.L + FA_NW * FA_QW - 1) / (FA_NW * FA_QW), a.H, B);
  launch_pdl(attn_tc_kernel<MODE, DHP, FA_NW>, grid, dim3(FA_NW * 32), FaCfg<DHP>::SMEM, st, a);
}

// mode AM_BF16 / AM_TF32X3; returns false for unsupported head dims.
// Short sequences (L <= 1024) take the key-split kernel, long ones the
// 32-query-tile kernel (better K/V reuse per CTA).
static inline bool launch_attn_tc(int mode, const AttnArgs& a, int B, cudaStream_t st) {
  if (a.dh % 8) return false;
  const bool ks = a.L <= 1024;
  if (mode == AM_BF16) {
    switch ((a.dh + 15) / 16 * 16) {
      case 32: ks ? launch_ks<AM_BF16, 32>(a, B, st) : launch_fa<AM_BF16, 32>(a, B, st); return true;
      case 64: ks ? launch_ks<AM_BF16, 64>(a, B, st) : launch_fa<AM_BF16, 64>(a, B, st); return true;
      case 80: ks ? launch_ks<AM_BF16, 80>(a, B, st) : launch_fa<AM_BF16, 80>(a, B, st); return true;
      case 128:  // the key-split stages would exceed 227 KB of smem at this width
        launch_fa<AM_BF16, 128>(a, B, st);
        return true;
      default: return false;
    }
  }
  switch (a.dh) {
    case 32: ks ? launch_ks<AM_TF32X3, 32>(a, B, st) : launch_fa<AM_TF32X3, 32>(a, B, st); return true;
    case 64: ks ? launch_ks<AM_TF32X3, 64>(a, B, st) : launch_fa<AM_TF32X3, 64>(a, B, st); return true;
    case 72: ks ? launch_ks<AM_TF32X3, 72>(a, B, st) : launch_fa<AM_TF32X3, 72>(a, B, st); return true;
    default: return false;
  }
}

}  // namespace ps
