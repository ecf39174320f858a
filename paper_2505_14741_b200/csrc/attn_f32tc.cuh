// tcgen05 attention for the fp32 predictor path (3xTF32, head_dim <= 64).
//
// softmax(Q K^T / sqrt(dh)) V for one (lane b, head, 128-query tile) per CTA,
// to ~fp32 accuracy: every operand x is split x = hi + lo (hi = x with the
// low 13 mantissa bits cleared, exactly representable in tf32; lo = x - hi,
// exact in fp32) and each product runs as lo*hi + hi*lo + hi*hi on
// `tcgen05.mma.kind::tf32` (the ~2^-22 lo*lo term is dropped), accumulated in
// fp32 in TMEM:
//
//   all 128 threads   Q (once), K_j, V_j: fp32 from the QKV GEMM's output
//                     [B*L, 3D] -> hi/lo split in registers -> shared memory
//                     in the 128-byte-swizzled K-major layout the MMA reads
//   warp 0 (elected)  S_j = Q K_j^T  (M=128, N=64, K=dh: 3 passes, SS form)
//                     O  += P_j V_j  (M=128, N=DHP, K=64: 3 passes; A = P
//                                     hi/lo from TMEM, B = V^T K-major smem)
//   thread r          query row r = TMEM lane r: tcgen05.ld S row, exact
//                     online softmax in fp32, P hi/lo rows via tcgen05.st
//
// TMEM (256 columns): S [0,64), P_hi [64,128), P_lo [128,192), O [192, 192+DHP).
// The key blocks of a query tile are split over a cluster of KS CTAs (CTA z
// runs blocks z, z+KS, ... with an exact online softmax that rescales O's
// row in TMEM when the row max moves); the KS partial (m, l, O) rows are
// merged over DSMEM in cluster-rank order, each CTA finishing 128/KS rows.
// Key blocks are 64 wide: DiT-S/2 (L = 256) runs 2 query tiles x 6 heads x
// KS = 4 -> 48 CTAs, one key block each. Fixed reduction order: results depend on KS only through the
// merge order, which is fixed per L.
// Replaces the mma.sync (HMMA) key-split kernel of attn_mma.cuh on the fp32
// path (the reference predictor contract: pkg/src/parastep/predictor.py:133).
#pragma once

#include "attn_fmha.cuh"

namespace ps {

constexpr int F3_BQ = 128, F3_BK = 64;
constexpr int F3_ATOM = 128 * 128;  // 128 rows x 128 B (32 fp32): one swizzle-atom column
constexpr int F3_THREADS = 256;     // warps 0-3: softmax rows; all 8 warps: loads and merge

template <int NA>  // head-dim atoms of 32 fp32: DHP = 32 * NA >= dh
struct F3Cfg {
  static constexpr int DHP = 32 * NA;
  static constexpr int TILE = NA * F3_ATOM;      // one 128-query operand copy (hi or lo)
  static constexpr int KT = NA * F3_BK * 128;     // one key-block copy: K, or V^T (DHP x BK)
  // smem: Q_hi Q_lo K_hi K_lo V_hi V_lo, then barriers
  static constexpr int BAR_OFF = 2 * TILE + 4 * KT;
  static constexpr int SMEM = BAR_OFF + 64 + 1024;
  static constexpr uint32_t T_S = 0, T_PHI = F3_BK, T_PLO = 2 * F3_BK, T_O = 3 * F3_BK;
  static constexpr uint32_t TMEM_COLS = 256;
  static_assert(T_O + DHP <= TMEM_COLS, "TMEM budget");
};

// tcgen05.mma kind::tf32 with A from tensor memory (TS form), elected lane
__device__ __forceinline__ void umma_tf32_ts_e(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ float f3_hi(float v) {
  return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
}

// ROWS rows x dh columns of fp32 at src (row stride ld floats; rows >= nvalid
// and columns >= dh read as 0) -> hi / lo copies in the SW128 K-major layout:
// atom a (columns [32a, 32a+32)) at a * ROWS * 128, row r at r * 128 B, 16-byte
// chunk c at ((c ^ (r & 7)) << 4) - the layout TMA SWIZZLE_128B produces.
// Split into a fetch (every global load of the tile issued at once, into
// registers) and a store (hi/lo split into smem), so the loads of the next
// key block are in flight while the current one is on the tensor core.
template <int NA, int ROWS>
struct F3Tile {
  static constexpr int CPR = NA * 8;                      // 16-byte chunks per row
  static constexpr int N = ROWS * CPR / F3_THREADS;       // chunks per thread
  static_assert(ROWS * CPR % F3_THREADS == 0, "whole chunks per thread");
  float4 v[N];
  __device__ __forceinline__ void fetch(const float* src, int64_t ld, int nvalid, int dh) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int q = threadIdx.x + i * F3_THREADS, r = q / CPR, d0 = 4 * (q % CPR);
      v[i] = (r < nvalid && d0 < dh) ? __ldg(reinterpret_cast<const float4*>(src + r * ld + d0))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  __device__ __forceinline__ void store(uint8_t* hi, uint8_t* lo) const {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int q = threadIdx.x + i * F3_THREADS, r = q / CPR, cc = q % CPR;
      const int off = (cc >> 3) * ROWS * 128 + r * 128 + (((cc & 7) ^ (r & 7)) << 4);
      const float4 h = make_float4(f3_hi(v[i].x), f3_hi(v[i].y), f3_hi(v[i].z), f3_hi(v[i].w));
      *reinterpret_cast<float4*>(hi + off) = h;
      *reinterpret_cast<float4*>(lo + off) =
          make_float4(v[i].x - h.x, v[i].y - h.y, v[i].z - h.z, v[i].w - h.w);
    }
  }
};

// V block (F3_BK keys x dh, same source layout) -> V^T hi / lo as the K-major
// B operand of P V: row n = head dim n, K = keys in atoms of 32 keys (128 B)
// at ka * DHP * 128 B. Lane = key (32 consecutive keys per warp pass), so a
// warp's scalar stores for one dim row fill 32 distinct banks. (A probe of
// kind::tf32 with V as an MN-major SW128 B operand, the bf16 kernel's form,
// accumulated nothing on B200, so V is transposed here instead.)
template <int NA>
struct F3VTile {
  static constexpr int DHP = 32 * NA;
  static constexpr int ITS = (F3_BK / 32) * (DHP / 4);  // (key group, dim quad) passes
  static constexpr int N = ITS / (F3_THREADS / 32);      // per warp
  static_assert(ITS % (F3_THREADS / 32) == 0, "whole passes per warp");
  float4 v[N];
  __device__ __forceinline__ void fetch(const float* src, int64_t ld, int nvalid, int dh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int it = warp + i * (F3_THREADS / 32);
      const int key = (it / (DHP / 4)) * 32 + lane, n0 = 4 * (it % (DHP / 4));
      v[i] = (key < nvalid && n0 < dh) ? __ldg(reinterpret_cast<const float4*>(src + key * ld + n0))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  __device__ __forceinline__ void store(uint8_t* hi, uint8_t* lo) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int it = warp + i * (F3_THREADS / 32);
      const int kb = it / (DHP / 4), n0 = 4 * (it % (DHP / 4));
      const float x[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
      const int cbase = kb * DHP * 128 + 4 * (lane & 3);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + j;
        const int off = cbase + n * 128 + ((((lane >> 2) ^ (n & 7))) << 4);
        const float h = f3_hi(x[j]);
        *reinterpret_cast<float*>(hi + off) = h;
        *reinterpret_cast<float*>(lo + off) = x[j] - h;
      }
    }
  }
};

template <int NA, int KS>
__global__ void __launch_bounds__(F3_THREADS, 1) fmha_f32_kernel(const __grid_constant__ AttnArgs p) {
  using C = F3Cfg<NA>;
  constexpr int DHP = C::DHP;
  extern __shared__ __align__(1024) uint8_t f3_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(f3_smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_hi = smem;
  uint8_t* q_lo = smem + C::TILE;
  uint8_t* k_hi = smem + 2 * C::TILE;
  uint8_t* k_lo = k_hi + C::KT;
  uint8_t* v_hi = k_hi + 2 * C::KT;
  uint8_t* v_lo = k_hi + 3 * C::KT;
  uint64_t* s_full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* pv_done = s_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);

  const int warp = threadIdx.x >> 5, r = threadIdx.x;
  // cluster of KS CTAs along x: CTA z of a query tile takes key blocks z, z + KS, ...
  const int z = KS > 1 ? (int)(blockIdx.x % KS) : 0;
  const int q0 = (blockIdx.x / KS) * F3_BQ, head = blockIdx.y, b = blockIdx.z;
  const int L = p.L, D = p.D, dh = p.dh;
  const int64_t ld = 3 * (int64_t)D;
  const float* base = p.qkv + (int64_t)b * L * ld + head * dh;
  const int nkb = (L + F3_BK - 1) / F3_BK;

  if (threadIdx.x == 0) {
    mbar_init(s_full, 1);
    mbar_init(pv_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  pdl_wait_and_release();

  constexpr uint32_t idS = make_idesc(KIND_TF32X3, 128, F3_BK);
  const float sl2 = p.scale * 1.4426950408889634f;
  float m_run = -INFINITY, l = 0.f;

  // Q and this CTA's first K / V block: every load in flight at once
  F3Tile<NA, F3_BQ> qt;
  F3Tile<NA, F3_BK> kt;
  F3VTile<NA> vt;
  qt.fetch(base + (int64_t)q0 * ld, ld, L - q0, dh);
  if (z < nkb) {
    kt.fetch(base + (int64_t)z * F3_BK * ld + D, ld, L - z * F3_BK, dh);
    vt.fetch(base + (int64_t)z * F3_BK * ld + 2 * D, ld, L - z * F3_BK, dh);
  }
  qt.store(q_hi, q_lo);
  int nloc = 0;  // key blocks this CTA ran
  for (int jb = z; jb < nkb; jb += KS, ++nloc) {
    const int j = nloc;  // local block index: barrier phases, first-block flags
    if (j > 0) {  // P_{j-1} V_{j-1} done: K/V smem, the P buffers and O are free
      mbar_wait(pv_done, (j - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    const int k0 = jb * F3_BK, valid = L - k0;
    kt.store(k_hi, k_lo);
    vt.store(v_hi, v_lo);
    if (jb + KS < nkb) {  // the next block's loads overlap this block's MMAs / softmax
      const int k1 = (jb + KS) * F3_BK;
      kt.fetch(base + (int64_t)k1 * ld + D, ld, L - k1, dh);
      vt.fetch(base + (int64_t)k1 * ld + 2 * D, ld, L - k1, dh);
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int k = 0; k < NA * 4; ++k) {  // K = 8 tf32 (32 B) per MMA; atom k / 4
        const uint64_t ko = (uint64_t)(2 * (k & 3));
        const int aq = (k >> 2) * F3_ATOM, ak = (k >> 2) * F3_BK * 128;
        const uint64_t qh = smem_desc_sw128(q_hi + aq) + ko, ql = smem_desc_sw128(q_lo + aq) + ko;
        const uint64_t kh = smem_desc_sw128(k_hi + ak) + ko, kl = smem_desc_sw128(k_lo + ak) + ko;
        umma_e<KIND_TF32X3>(tmem + C::T_S, ql, kh, idS, k > 0 ? 1u : 0u);
        umma_e<KIND_TF32X3>(tmem + C::T_S, qh, kl, idS, 1u);
        umma_e<KIND_TF32X3>(tmem + C::T_S, qh, kh, idS, 1u);
      }
      umma_commit_e(s_full);
    }
    if (warp < 4) {  // softmax: thread r <-> query row r <-> TMEM lane r
      mbar_wait(s_full, j & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // ---- exact online softmax of row r over this key block
      float sv[F3_BK];
#pragma unroll
      for (int c = 0; c < F3_BK / 32; ++c) tmem_ld32(tmem + C::T_S + lane_off + c * 32, sv + c * 32);
      tmem_ld_wait();
      if (valid < F3_BK) {
#pragma unroll
        for (int i = 0; i < F3_BK; ++i)
          if (i >= valid) sv[i] = -INFINITY;
      }
      float pm[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) pm[i] = -INFINITY;
#pragma unroll
      for (int i = 0; i < F3_BK; ++i) pm[i & 7] = fmaxf(pm[i & 7], sv[i]);
      const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                             fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      const float m_new = fmaxf(m_run, mx * sl2);
      const float f = exp2f(m_run - m_new);  // 0 on the first block (m_run = -inf)
      m_run = m_new;
      float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < F3_BK; ++i) {
        const float e = fast_exp2(fmaf(sv[i], sl2, -m_new));  // masked keys: exp2(-inf) = 0
        ps[i & 3] += e;
        sv[i] = e;
      }
      l = fmaf(l, f, (ps[0] + ps[1]) + (ps[2] + ps[3]));
      if (j > 0 && __any_sync(0xffffffffu, f != 1.f)) {  // O row *= f (P_{j-1} V_{j-1} landed)
#pragma unroll
        for (int c = 0; c < DHP / 32; ++c) {
          float o[32];
          tmem_ld32(tmem + C::T_O + lane_off + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= f;
          tmem_st32(tmem + C::T_O + lane_off + c * 32, o);
        }
      }
#pragma unroll
      for (int c = 0; c < F3_BK / 32; ++c) {
        float h[32], lo[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          h[i] = f3_hi(sv[c * 32 + i]);
          lo[i] = sv[c * 32 + i] - h[i];
        }
        tmem_st32(tmem + C::T_PHI + lane_off + c * 32, h);
        tmem_st32(tmem + C::T_PLO + lane_off + c * 32, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // B = V^T, K-major: atom ka (keys [32ka, 32ka+32)) at ka * DHP * 128 B
      constexpr uint32_t idPV = make_idesc(KIND_TF32X3, 128, DHP);
#pragma unroll
      for (int k = 0; k < F3_BK / 8; ++k) {  // 8 keys = 8 TMEM columns of P = 32 B of V^T
        const uint64_t ko = (uint64_t)(2 * (k & 3));
        const int ao = (k >> 2) * DHP * 128;
        const uint64_t vh = smem_desc_sw128(v_hi + ao) + ko, vl = smem_desc_sw128(v_lo + ao) + ko;
        const uint32_t acc = (j | k) ? 1u : 0u;
        umma_tf32_ts_e(tmem + C::T_O, tmem + C::T_PLO + 8 * k, vh, idPV, acc);
        umma_tf32_ts_e(tmem + C::T_O, tmem + C::T_PHI + 8 * k, vl, idPV, 1u);
        umma_tf32_ts_e(tmem + C::T_O, tmem + C::T_PHI + 8 * k, vh, idPV, 1u);
      }
      umma_commit_e(pv_done);
    }
  }
  // ---- partial (m, l, O) of row r -> smem (Q/K regions are free: every MMA
  // has completed); with KS > 1 the cluster merges its partials over DSMEM
  constexpr int PST = DHP + 4;  // row stride (floats): O[DHP], m, l
  float* part = reinterpret_cast<float*>(smem);
  if (nloc > 0) {
    mbar_wait(pv_done, (nloc - 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if (warp < 4) {
#pragma unroll
    for (int c = 0; c < DHP / 32; ++c) {
      float o[32];
      tmem_ld32(tmem + C::T_O + lane_off + c * 32, o);
      tmem_ld_wait();
#pragma unroll
      for (int g = 0; g < 8; ++g)
        *reinterpret_cast<float4*>(part + r * PST + c * 32 + 4 * g) =
            nloc > 0 ? make_float4(o[4 * g], o[4 * g + 1], o[4 * g + 2], o[4 * g + 3])
                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    *reinterpret_cast<float4*>(part + r * PST + DHP) = make_float4(m_run, l, 0.f, 0.f);
  }
  if (KS > 1)
    cluster_sync_all();
  else
    __syncthreads();
  // CTA z writes rows [z * 128 / KS, (z + 1) * 128 / KS): the partials merged
  // in cluster-rank order, O / l in the proj GEMM's operand format, with
  // consecutive threads on consecutive 4-dim groups of a row
  constexpr int RPC = F3_BQ / KS, G4 = DHP / 4;
  for (int it = threadIdx.x; it < RPC * G4; it += F3_THREADS) {
    const int rr = z * RPC + it / G4, d = 4 * (it % G4);
    const int q = q0 + rr;
    if (q >= L || d >= dh) continue;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float lsum = 0.f;
    if (KS == 1) {
      acc = *reinterpret_cast<const float4*>(part + rr * PST + d);
      lsum = part[rr * PST + DHP + 1];
    } else {
      float mz[KS], lz[KS];
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < KS; ++c) {
        const float4 ml = ld_dsmem_f4(part + rr * PST + DHP, (uint32_t)c);
        mz[c] = ml.x;
        lz[c] = ml.y;
        mx = fmaxf(mx, ml.x);
      }
#pragma unroll
      for (int c = 0; c < KS; ++c) {
        const float w = lz[c] > 0.f ? exp2f(mz[c] - mx) : 0.f;  // CTAs without keys: 0
        const float4 oc = ld_dsmem_f4(part + rr * PST + d, (uint32_t)c);
        acc.x = fmaf(w, oc.x, acc.x);
        acc.y = fmaf(w, oc.y, acc.y);
        acc.z = fmaf(w, oc.z, acc.z);
        acc.w = fmaf(w, oc.w, acc.w);
        lsum = fmaf(w, lz[c], lsum);
      }
    }
    const float inv = 1.f / lsum;
    const float4 v = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    const int64_t o = ((int64_t)b * L + q) * D + head * dh + d;
    if (p.out_hi) {
      const float4 h = make_float4(f3_hi(v.x), f3_hi(v.y), f3_hi(v.z), f3_hi(v.w));
      *reinterpret_cast<float4*>(p.out_hi + o) = h;
      *reinterpret_cast<float4*>(p.out_lo + o) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z,
                                                             v.w - h.w);
    }
    if (p.out_f32) *reinterpret_cast<float4*>(p.out_f32 + o) = v;
  }
  if (KS > 1) cluster_sync_all();  // peers may still read this CTA's partials
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::TMEM_COLS));
  }
}

}  // namespace ps
