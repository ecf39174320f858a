// tcgen05 flash attention, bf16 operands (head_dim <= 128).
//
// softmax(Q K^T / sqrt(dh)) V for one (lane b, head, NQ x 128-query tiles)
// per CTA, Q/K/V read by TMA straight out of the QKV GEMM's bf16 output
// [B*L, 3D] (128-byte swizzled boxes of 128 tokens x 64 dims); scores, the
// bf16 probabilities and the output accumulator all live in TMEM:
//
//   TMA warp (1 lane)   Q once, then K_j/V_j into a 2-3 stage ring
//   MMA warp (elected)  S_j = Q K_j^T  (M=128, N=128, K=DH; A, B from smem)
//                       O  += P_j V_j  (M=128, N=DH, K=128; A = P from TMEM,
//                                       B = V MN-major from smem)
//   4 softmax warps     thread r owns query row r (TMEM lane r): tcgen05.ld
//   per query tile      S row -> exp2 -> bf16 P row, tcgen05.st into TMEM
//
// The next block's scores are issued as soon as the softmax has read S out
// of TMEM (NQ = 2: s_free, mid exp pass; NQ = 1: double-buffered S), ahead
// of P V, so the softmax never waits on its own P V. Keeping P in TMEM takes
// the P writes and the A-operand reads of P V off shared memory, which was
// the tensor core's feed bottleneck. Online softmax with a lazy rescale: a
// row's reference max only moves when the block max exceeds it by more than
// 2^8 (then O's row is rescaled in TMEM, after P_{j-1} V_{j-1} has landed);
// otherwise p = exp2(s - m_ref) <= 256, exact in fp32 and safe in bf16. A
// fixed share of the exps runs on the FMA pipe (poly_exp2) to unload MUFU.
// The final O / l goes out in the proj GEMM's bf16 operand layout. All
// reductions run in a fixed order: results do not depend on the grid.
#pragma once

#include "attn_fmha.h"
#include "attn_mma.cuh"
#include "gemm_tc.cuh"

namespace ps {

constexpr int FM_BQ = 128, FM_BK = 128;
// TMEM columns: S buffers [0, 256), O [256, 256 + NQ*DH) (NQ*DH <= 128), and
// the bf16 P buffers (64 columns each) at [384, 512)
constexpr int FM_TP = 384;
constexpr int FM_TILE = 128 * 128;  // bytes of one 128-row x 128-byte (64 bf16) box

// DH = padded head width in smem/TMEM (64, or 128 for head_dim 72..128):
// NA = DH/64 swizzle atoms along the head dim per Q/K/V tile.
// NQ = 128-query tiles per CTA sharing each K/V block:
//   NQ = 1: S and P double-buffered (S0 [0,128) S1 [128,256), O [256,256+DH),
//           P0/P1 [384, 512)); short sequences (more CTAs)
//   NQ = 2: two softmax warpgroups (tile t: S_t [128t, 128t+128), O_t
//           [256 + 64t, ...), P_t [384 + 64t, ...)), one S and one P buffer per
//           tile; the tensor core runs tile 1's MMAs under tile 0's softmax
template <int DH, int NQ>
struct FmCfg {
  static constexpr int NA = DH / 64;
  static constexpr int STAGES = DH == 64 ? 3 : 2;
  static constexpr int THREADS = (4 * NQ + 2) * 32;
  static constexpr int Q_OFF = 0;
  static constexpr int KV_OFF = NQ * NA * FM_TILE;  // stage s: K at +2s*NA*TILE, V at +(2s+1)*NA*TILE
  static constexpr int BAR_OFF = KV_OFF + 2 * STAGES * NA * FM_TILE;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr uint32_t TMEM_COLS = 512;
  static_assert(NQ == 1 || DH == 64, "two query tiles only for 64-wide heads (smem)");
};

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]),
      "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]),
      "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// exp2 on the FMA / ALU pipes: x = j + f with j = rint(x) (magic-number
// round), 2^f by a degree-3 minimax polynomial on [-0.5, 0.5] (max relative
// error 1.0e-4, far below P's bf16 rounding), 2^j added to the exponent
// field. x is clamped at -127 so -inf (masked keys) gives exactly +0. Used
// for a fixed share of the exps (POLY of every 4 pairs) to take load off the
// MUFU unit (16 ex2 / clk / SM).
__device__ __forceinline__ float poly_exp2(float x) {
  x = fmaxf(x, -127.f);
  const float r = x + 12582912.f;  // 1.5 * 2^23
  const float f = x - (r - 12582912.f);
  const float q = fmaf(fmaf(fmaf(0.0550089292f, f, 0.242210984f), f, 0.693282902f), f, 1.f);
  return __int_as_float(__float_as_int(q) + (__float_as_int(r) << 23));
}

// Blackwell packed fp32 pairs (FFMA2 / FADD2) and the 3-input max (FMNMX3):
// the softmax's per-element ALU work in half the issue slots. Lane-wise the
// same IEEE operations as fmaf / + / fmaxf.
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(f2_pack(a.x, a.y)), "l"(f2_pack(b.x, b.y)), "l"(f2_pack(c.x, c.y)));
  return f2_unpack(r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a.x, a.y)), "l"(f2_pack(b.x, b.y)));
  return f2_unpack(r);
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// poly_exp2 on a pair (FFMA2 / FADD2 Horner): lane-wise identical to poly_exp2
__device__ __forceinline__ float2 poly_exp2x2(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 mg = make_float2(12582912.f, 12582912.f);
  const float2 r = fadd2(x, mg);
  const float2 f = fadd2(x, make_float2(-(r.x - 12582912.f), -(r.y - 12582912.f)));
  float2 q = ffma2(make_float2(0.0550089292f, 0.0550089292f), f,
                   make_float2(0.242210984f, 0.242210984f));
  q = ffma2(q, f, make_float2(0.693282902f, 0.693282902f));
  q = ffma2(q, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(r.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(r.y) << 23)));
}

#ifdef FMHA_STAMPS
__device__ long long g_fm_ts[9][32][4];
#define FM_TS(role, j, k) \
  do { if (blockIdx.x == 0 && blockIdx.y == 0 && (j) < 32) g_fm_ts[role][j][k] = clock64(); } while (0)
#else
#define FM_TS(role, j, k) do {} while (0)
#endif

template <int DH, int NQ, int POLY>
__global__ void __launch_bounds__(FmCfg<DH, NQ>::THREADS, 1)
    fmha_tc_kernel(const __grid_constant__ CUtensorMap mapQKV, const __grid_constant__ FmhaArgs p) {
  using C = FmCfg<DH, NQ>;
  constexpr int W_TMA = 4 * NQ, W_MMA = 4 * NQ + 1;
  constexpr int NA = C::NA, FM_STAGES = C::STAGES, FM_Q_OFF = C::Q_OFF, FM_KV_OFF = C::KV_OFF,
                FM_BAR_OFF = C::BAR_OFF;
  constexpr uint32_t FM_TMEM_COLS = C::TMEM_COLS;
  extern __shared__ __align__(1024) uint8_t fm_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(fm_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FM_BAR_OFF);
  uint64_t* q_full = bars;                    // 1
  uint64_t* kv_full = bars + 1;               // FM_STAGES
  uint64_t* kv_empty = kv_full + FM_STAGES;   // FM_STAGES
  uint64_t* s_full = kv_empty + FM_STAGES;    // 2
  uint64_t* p_full = s_full + 2;              // 2
  uint64_t* pv_done = p_full + 2;             // 2
  uint64_t* s_free = pv_done + 2;             // 2 (NQ = 2: S_t read out of TMEM)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_free + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * FM_BQ * NQ, head = blockIdx.y, b = blockIdx.z;
  const int L = p.L;
  const int nkb = (L + FM_BK - 1) / FM_BK;
  const int row_base = b * L;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mapQKV);
    mbar_init(q_full, 1);
    for (int s = 0; s < FM_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {  // NQ = 1: buffer j & 1; NQ = 2: query tile
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&pv_done[i], 1);
      mbar_init(&s_free[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(FM_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_wait_and_release();

  if (warp == W_TMA) {
    if (lane == 0) {
      // ---------------- TMA producer
      // column of (which, head, atom a) in the [rows, 3*H*DH] operand
      const int hc = head * DH, wstride = p.H * DH;
      mbar_expect_tx(q_full, NQ * NA * FM_TILE);
      for (int t = 0; t < NQ; ++t)
        for (int a = 0; a < NA; ++a)
          tma_load_2d(smem + FM_Q_OFF + (t * NA + a) * FM_TILE, &mapQKV, q_full, hc + 64 * a,
                      row_base + q0 + t * FM_BQ);
      for (int j = 0; j < nkb; ++j) {
        const int s = j % FM_STAGES;
        mbar_wait(&kv_empty[s], ((j / FM_STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[s], 2 * NA * FM_TILE);
        uint8_t* st = smem + FM_KV_OFF + 2 * s * NA * FM_TILE;
        for (int a = 0; a < NA; ++a) {
          tma_load_2d(st + a * FM_TILE, &mapQKV, &kv_full[s], wstride + hc + 64 * a,
                      row_base + j * FM_BK);
          tma_load_2d(st + (NA + a) * FM_TILE, &mapQKV, &kv_full[s], 2 * wstride + hc + 64 * a,
                      row_base + j * FM_BK);
        }
      }
    }
  } else if (warp == W_MMA) {
    {
      // ---------------- MMA issuer: the whole warp runs the loop (descriptors
      // in uniform registers), one elected lane issues each tcgen05 op
      constexpr uint32_t idS = make_idesc(KIND_BF16, 128, 128);
      // the zero-padded head dims beyond dh do no tensor work: S runs
      // ceil(dh/16) K-steps, P V an N of round_up(dh, 16) (DiT-XL/2's 72 -> 80
      // of the 128-wide operand); O's columns past that are never stored
      const int kdh = (p.dh + 15) / 16;
      const uint32_t idPV = make_idesc(KIND_BF16, 128, 16 * kdh) | (1u << 16);  // B (V) MN-major
      // S_t(j) = Q_t K_j^T into S buffer `sb`
      auto issue_s = [&](int t, int j, int sb) {
        const int s = j % FM_STAGES;
        mbar_wait(&kv_full[s], (j / FM_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* kt = smem + FM_KV_OFF + 2 * s * NA * FM_TILE;
        const uint8_t* qt = smem + FM_Q_OFF + t * NA * FM_TILE;
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {  // atom k/4, +32 B along K inside it
          if (k >= kdh) break;
          const uint64_t qd = smem_desc_sw128(qt + (k >> 2) * FM_TILE) + 2 * (k & 3);
          const uint64_t kd = smem_desc_sw128(kt + (k >> 2) * FM_TILE) + 2 * (k & 3);
          umma_e<KIND_BF16>(tmem + 128 * sb, qd, kd, idS, k > 0 ? 1u : 0u);
        }
        umma_commit_e(&s_full[sb]);
      };
      // O_t += P(buffer pb) V_j, once P has been written (p_full[pb], parity par)
      auto issue_pv = [&](int t, int j, int pb, int par) {
        mbar_wait(&p_full[pb], par);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int s = j % FM_STAGES;
        const uint32_t tP = tmem + FM_TP + pb * 64;
        // V: MN-major, NA atoms of 64 dims at FM_TILE stride (LBO), 8-key groups at 1 KB (SBO)
        const uint64_t vd = (smem_desc_sw128(smem + FM_KV_OFF + (2 * s + 1) * NA * FM_TILE) &
                             ~(0x3FFFull << 16)) |
                            ((uint64_t)(FM_TILE >> 4) << 16);
        const uint32_t tO = tmem + 256 + (NQ == 1 ? 0 : t * DH);
#pragma unroll
        for (int k = 0; k < FM_BK / 16; ++k)  // P: 16 keys = 8 TMEM columns; V: 16 keys = 2048 B
          umma_ts_e(tO, tP + 8 * k, vd + (uint64_t)(k * 2048 >> 4), idPV, (j | k) ? 1u : 0u);
      };
      mbar_wait(q_full, 0);
      if constexpr (NQ == 1) {
        issue_s(0, 0, 0);
        if (nkb > 1) issue_s(0, 1, 1);
        for (int j = 0; j < nkb; ++j) {
          issue_pv(0, j, j & 1, (j >> 1) & 1);
          umma_commit_e(&kv_empty[j % FM_STAGES]);
          umma_commit_e(&pv_done[j & 1]);
          if (j + 2 < nkb) issue_s(0, j + 2, j & 1);
        }
      } else {
        // S_t(j+1) goes in as soon as the softmax has read S_t(j) out of TMEM
        // (s_free, mid exp pass), ahead of P_t(j) V_j: the next block's
        // scores are ready when the softmax finishes this one
        issue_s(0, 0, 0);
        issue_s(1, 0, 1);
        for (int j = 0; j < nkb; ++j) {
          if (j + 1 < nkb) {
            mbar_wait(&s_free[0], j & 1);
            issue_s(0, j + 1, 0);
          }
          FM_TS(8, j, 0);
          issue_pv(0, j, 0, j & 1);
          umma_commit_e(&pv_done[0]);
          FM_TS(8, j, 1);
          if (j + 1 < nkb) {
            mbar_wait(&s_free[1], j & 1);
            issue_s(1, j + 1, 1);
          }
          FM_TS(8, j, 2);
          issue_pv(1, j, 1, j & 1);
          umma_commit_e(&kv_empty[j % FM_STAGES]);
          umma_commit_e(&pv_done[1]);
          FM_TS(8, j, 3);
        }
      }
    }
  } else {
    // ---------------- softmax warps: tile t, thread r <-> query row r <-> TMEM lane r
    const int t = warp >> 2;
    const int r = threadIdx.x & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tO = tmem + 256 + (NQ == 1 ? 0 : t * DH);
    // NQ = 1: buffers alternate per block (phase per pair of blocks);
    // NQ = 2: one buffer per tile (phase per block)
    auto buf = [&](int j) { return NQ == 1 ? (j & 1) : t; };
    auto par = [&](int j) { return NQ == 1 ? ((j >> 1) & 1) : (j & 1); };
    const float sl2 = p.scale_log2;
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(&s_full[buf(j)], par(j));
      if (lane == 0) FM_TS(warp, j, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // Row max. NQ = 1: the whole 128-column S row is loaded once and kept in
      // registers for the exp pass; NQ = 2 (register-limited, 10 warps):
      // streamed from TMEM 64 columns at a time and reloaded for the exp pass.
      // Reductions use 8 independent partial maxima / 4 partial sums (no
      // 128-long dependency chain); the order is fixed, so results do not
      // depend on NQ.
      const uint32_t srow = tmem + 128 * buf(j) + lane_off;
      const int valid = L - j * FM_BK;  // keys of this block inside the lane
      constexpr int CH = NQ == 1 ? FM_BK : 64;  // columns per TMEM load group
      float sv[CH];
      float pm[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) pm[i] = -INFINITY;
#pragma unroll
      for (int g = 0; g < FM_BK / CH; ++g) {
#pragma unroll
        for (int c = 0; c < CH / 32; ++c) tmem_ld32(srow + g * CH + c * 32, sv + c * 32);
        tmem_ld_wait();
        if (valid < FM_BK) {  // last block only: keys past the lane -> -inf (p = 0)
#pragma unroll
          for (int i = 0; i < CH; ++i)
            if (g * CH + i >= valid) sv[i] = -INFINITY;
        }
#pragma unroll
        for (int i = 0; i < CH; i += 2) pm[(i >> 1) & 7] = fmax3(pm[(i >> 1) & 7], sv[i], sv[i + 1]);
      }
      const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                             fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      const float m_new = mx * sl2;
      if (j == 0) {
        m_ref = m_new;
      } else {
        const bool need = m_new > m_ref + 8.f;
        if (__any_sync(0xffffffffu, need)) {
          // O's row must hold P_{j-1} V_{j-1} before it is rescaled
          mbar_wait(&pv_done[buf(j - 1)], par(j - 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const float m_tgt = need ? m_new : m_ref;
          const float f = fast_exp2(m_ref - m_tgt);
          l *= f;
          m_ref = m_tgt;
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            float o[32];
            tmem_ld32(tO + lane_off + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= f;
            tmem_st32(tO + lane_off + c * 32, o);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
      if (lane == 0) FM_TS(warp, j, 1);
      // the P buffer was last read by P V of block j-2 (NQ = 1) / j-1 (NQ = 2)
      if (NQ == 1 && j >= 2) mbar_wait(&pv_done[buf(j)], par(j - 2));
      if (NQ == 2 && j >= 1) mbar_wait(&pv_done[t], par(j - 1));
      if (lane == 0) FM_TS(warp, j, 2);
      const uint32_t prow = tmem + FM_TP + buf(j) * 64 + lane_off;  // bf16 pairs
      float2 ps[4];  // per pair slot q: (even key, odd key) partial row sums
#pragma unroll
      for (int q = 0; q < 4; ++q) ps[q] = make_float2(0.f, 0.f);
      const float2 sl2x2 = make_float2(sl2, sl2), nm2 = make_float2(-m_ref, -m_ref);
#pragma unroll
      for (int g = 0; g < FM_BK / CH; ++g) {  // exp2, row sum, bf16 P row
        if (NQ != 1) {
#pragma unroll
          for (int c = 0; c < CH / 32; ++c) tmem_ld32(srow + g * CH + c * 32, sv + c * 32);
          tmem_ld_wait();
          if (g == FM_BK / CH - 1) {  // S_t fully read: the MMA warp may overwrite it
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_free[t]);
          }
          if (valid < FM_BK) {
#pragma unroll
            for (int i = 0; i < CH; ++i)
              if (g * CH + i >= valid) sv[i] = -INFINITY;
          }
        }
        float pk[CH / 2];  // bf16 pairs of this group, column (key / 2)
#pragma unroll
        for (int h = 0; h < CH / 8; ++h) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i0 = h * 8 + 2 * q;  // masked keys hold -inf: exp2 -> +0
            const float2 x = ffma2(make_float2(sv[i0], sv[i0 + 1]), sl2x2, nm2);
            const float2 pp = q < POLY ? poly_exp2x2(x)
                                       : make_float2(fast_exp2(x.x), fast_exp2(x.y));
            ps[q] = fadd2(ps[q], pp);
            pk[i0 / 2] = __uint_as_float(pack_bf16(pp.x, pp.y));
          }
        }
#pragma unroll
        for (int c = 0; c < CH / 64; ++c) tmem_st32(prow + g * (CH / 2) + c * 32, pk + c * 32);
      }
      const float rs = ((ps[0].x + ps[0].y) + (ps[1].x + ps[1].y)) +
                       ((ps[2].x + ps[2].y) + (ps[3].x + ps[3].y));
      l += rs;
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&p_full[buf(j)]);
      if (lane == 0) FM_TS(warp, j, 3);
    }
    // ---------------- epilogue: O / l -> bf16 [B*L, D]
    mbar_wait(&pv_done[buf(nkb - 1)], par(nkb - 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const float inv = 1.f / l;
    const int q = q0 + t * FM_BQ + r;
    const bool ok = q < L;
    __nv_bfloat16* orow = p.out_bf16 + (int64_t)(row_base + q) * p.D + head * p.dh;
#pragma unroll
    for (int c = 0; c < DH / 32; ++c) {
      float o[32];
      tmem_ld32(tO + lane_off + c * 32, o);
      tmem_ld_wait();
      if (ok) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (c * 32 + 8 * q >= p.dh) break;  // padded dims (dh % 8 == 0)
          uint4 u;
          u.x = pack_bf16(o[8 * q] * inv, o[8 * q + 1] * inv);
          u.y = pack_bf16(o[8 * q + 2] * inv, o[8 * q + 3] * inv);
          u.z = pack_bf16(o[8 * q + 4] * inv, o[8 * q + 5] * inv);
          u.w = pack_bf16(o[8 * q + 6] * inv, o[8 * q + 7] * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + 8 * q) = u;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(FM_TMEM_COLS));
  }
}

}  // namespace ps
