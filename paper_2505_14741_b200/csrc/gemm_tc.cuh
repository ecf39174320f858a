// tcgen05 tensor-core GEMM for the DiT predictor (sm_100a).
//
//   C[M, N] = A[M, K] x W[K, N] + bias, fused DiT epilogues (gemm_simt.cuh Epi)
//
// Operands are K-major in HBM: A (activations) row-major [M][K] exactly as
// the producing kernel (LN-modulate / attention / GELU epilogue) writes it;
// W is transposed once at load into [N][K]. Per CTA tile 128 x BN:
//   warp 0 (1 thread)  TMA producer: 128-byte-swizzled K slabs -> smem ring
//   warp 1 (1 thread)  MMA issuer:   tcgen05.mma, accumulator in TMEM
//   warp 2             TMEM allocator
//   warps 0-3          epilogue:     tcgen05.ld -> registers -> fused store
// Two precisions:
//   KIND_BF16  kind::f16, bf16 x bf16 -> fp32 (configs[2], DiT-XL/2 bf16)
//   KIND_TF32X3 kind::tf32 with the 3-pass split a = a_hi + a_lo:
//              a_hi*b_hi + a_hi*b_lo + a_lo*b_hi  (~fp32 accuracy for the
//              1e-4 fp32 path, configs[1]); producers write a_hi/a_lo.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <type_traits>
#include <vector>

#include "gemm_simt.cuh"

namespace ps {

enum { KIND_BF16 = 0, KIND_TF32X3 = 1 };

struct TcOperand {
  float* f32 = nullptr;
  __nv_bfloat16* bf16 = nullptr;
  float* hi = nullptr;
  float* lo = nullptr;
  int rows = 0, cols = 0;
  // A maps (128-row boxes): bf16 or tf32-hi / tf32-lo. (Entries 1-2 held
  // 64/32-row boxes for an A-tile TMA multicast across N-tile CTAs, which
  // measured slower at every DiT/U-Net shape and was removed.)
  CUtensorMap map_main[3];
  CUtensorMap map_lo[3];
};

struct TcActs {
  TcOperand a, o, hid;
  std::vector<void*> owned;
};

struct TcLayer {
  int K, N;
  void* w_main = nullptr;  // bf16 [N][K] or tf32-hi fp32 [N][K]
  void* w_lo = nullptr;    // tf32-lo fp32 [N][K]
  // B operand maps per N-tile width (index 0: 32 rows, 1: 64, 2: 128); *_lo
  // are the tf32-lo copies of the 3xTF32 path
  CUtensorMap map_b[3], map_blo[3];
  int splits = 1;  // split-K factor, fixed per layer (independent of M: batch == single bitwise)
  int bn = 64;     // planned N-tile width at ref_rows
  int ref_rows = 0;
};

struct TcWeights {
  std::vector<TcLayer> layers;
  int precision = 0;
};

constexpr int TC_BM = 128;
constexpr int TC_THREADS = 128;
constexpr int TC_SMEM_BUDGET = 200 * 1024;  // stage ring per CTA

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// K-major, 128-byte swizzle smem matrix descriptor (tcgen05 "shared memory
// descriptor"): start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major,
// 1), SBO>>4 [32,46) = 1024 B between 8-row groups, version 1 at [46,48),
// layout SWIZZLE_128B = 2 at [61,64).
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= 1ull << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

// instruction descriptor: D fp32, A/B format, both K-major, N>>3, M>>4
__host__ __device__ constexpr uint32_t make_idesc(int kind, int M, int N) {
  const uint32_t fmt = kind == KIND_BF16 ? 1u : 2u;  // BF16 = 1, TF32 = 2
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

template <int KIND>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                     uint32_t idesc, uint32_t accumulate) {
  if constexpr (KIND == KIND_BF16) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}

// Warp-wide variants: every lane of the issuing warp executes them (so the
// descriptor arithmetic stays in uniform registers) and one elected lane
// issues the instruction.
template <int KIND>
__device__ __forceinline__ void umma_e(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  if constexpr (KIND == KIND_BF16) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}

__device__ __forceinline__ void mbar_arrive_e(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// (A operand read from tensor memory: tmem_a = 128 lanes x 16 bf16 = 8 columns)
__device__ __forceinline__ void umma_ts_e(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit_e(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%"
      "15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ------------------------------------------------------------------ kernel
template <int KIND, int BN>
struct TcCfg {
  static constexpr int BK_BYTES = 128;
  static constexpr int ESZ = KIND == KIND_BF16 ? 2 : 4;
  static constexpr int BK = BK_BYTES / ESZ;            // K elements per stage
  static constexpr int UK = KIND == KIND_BF16 ? 16 : 8;  // K per MMA
  static constexpr int A_BYTES = TC_BM * BK_BYTES;
  static constexpr int B_BYTES = BN * BK_BYTES;
  static constexpr int NOPS = KIND == KIND_BF16 ? 1 : 2;  // main (+lo) copies
  static constexpr int STAGE_BYTES = NOPS * (A_BYTES + B_BYTES);
  // 4 stages (3 for tf3x BN=128: 3 x 64 KB). Measured: deeper rings (up to
  // 10) do not speed up the small-M mainloop, which is bound by per-SM TMA
  // ingest (~70 GB/s/SM), and 6 stages cost the large-M GEMMs ~25%
  // (CogVideoX fc1 753 -> 959 us, same box A/B)
  static constexpr int STAGES_FIT = TC_SMEM_BUDGET / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT < 3 ? 3 : (STAGES_FIT > 4 ? 4 : STAGES_FIT);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

// Deterministic split-K. A layer's K range is cut into S segments (S fixed
// per layer, see tc_prepare) and the result is always
//     acc = ((seg_0 + seg_1) + seg_2) + ...      (each seg_s accumulated in TMEM)
// whichever way the segments are executed, so a row's bits never depend on
// the batch:
//   cluster == S  small M (few tiles): the S segment-CTAs of a tile form a
//                 thread-block cluster (1, 1, S); each parks its fp32 partial
//                 tile in its own drained smem ring, and after a cluster
//                 barrier CTA z reduces rows [z*128/S, (z+1)*128/S) over DSMEM
//                 in segment order and runs the fused epilogue;
//   cluster == 1  large M: one CTA runs all S segments into S TMEM
//                 accumulators and adds them in the same order.
struct TcSplit {
  int splits;   // S: K segments (fixed per layer)
  int cluster;  // SC: CTAs along K per tile (1 = all segments in one CTA; S/SC each)
  int seg[9];   // K-block bounds of the segments: segment g = [seg[g], seg[g+1])
};
// cluster dims (1, 1, cluster): rank = z

// DSMEM load of a peer's partial tile. Not volatile / no memory clobber: the
// data is immutable between the two cluster barriers that bracket the
// reduction (those carry the ordering), so the compiler may batch and
// hoist these loads across iterations.
__device__ __forceinline__ float4 ld_dsmem_f4(const float* local, uint32_t cta) {
  uint32_t remote;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(cta));
  float4 v;
  asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "r"(remote));
  return v;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// DSMEM split-K reduction: float4 loads in flight per thread per pass
// (measured 4 / 8 / 16: 4 best end to end - DiT-S 38.7 vs 39.7 ms, U-Net
// 709 vs 728 / 746 ms; profiles/r1d_epilogue_variants.txt)
constexpr int TC_REDUCE_LOADS = 4;

// Coalesced epilogue for one warp's 32 accumulator rows x NC columns that the
// warp has staged row-major in smem (stride EST floats): written back row by
// row with consecutive lanes on consecutive 4-column groups, so every store
// (and the residual / gate reads of EPI_RESID / EPI_ADD) is a contiguous run
// of up to 512 B. The TMEM layout alone (thread = row) would make each warp
// instruction touch 32 rows at once - measured 6-20x slower for the gated
// residual epilogue at CogVideoX shape, where the residual stream exceeds L2.
template <int NC, int EST>
__device__ __forceinline__ void warp_store_rows(const Epi& e, const float* stg, int row0, int col0,
                                                int M, int N, int lane, int nrows = 32) {
  static_assert(NC % 4 == 0 && NC <= 128, "one float4 column group per lane and row");
  constexpr int LPR = NC / 4 < 32 ? NC / 4 : 32;  // lanes per row
  constexpr int RPP = 32 / LPR;                   // rows per pass
  if ((e.mode == EPI_RESID || (e.mode == EPI_ADD && !e.pad_DH)) && (N & 3) == 0) {
    // Read-modify-write modes: the residual is updated in place, so the
    // compiler cannot hoist row r+1's loads above row r's store - issue RB
    // rows of loads first (memory-level parallelism), then finish them. Same
    // arithmetic, in the same order, as epi_store4 / epi_store16.
    constexpr int RB = 8;
    const int c4 = (lane % LPR) * 4, col = col0 + c4;
    if (c4 >= NC || col >= N) return;
    const float4 bb = e.bias ? *reinterpret_cast<const float4*>(e.bias + col)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    const bool resid_mode = e.mode == EPI_RESID;
#pragma unroll 1
    for (int r0 = 0; r0 < nrows; r0 += RPP * RB) {
      float4 ga[RB], rb[RB];
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int r = r0 + i * RPP + lane / LPR, grow = row0 + r;
        ga[i] = rb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (grow >= M || r >= nrows) continue;
        const int64_t base = (int64_t)grow * N + col;
        if (resid_mode)
          ga[i] = *reinterpret_cast<const float4*>(gate_row(e, grow) + col);
        else if (e.vec)
          ga[i] = *reinterpret_cast<const float4*>(e.vec + lane_row(e, grow) * e.vec_stride + col);
        if (e.resid) rb[i] = *reinterpret_cast<const float4*>(e.resid + base);
      }
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int r = r0 + i * RPP + lane / LPR, grow = row0 + r;
        if (grow >= M || r >= nrows) continue;
        const int64_t base = (int64_t)grow * N + col;
        const float4 a = *reinterpret_cast<const float4*>(stg + r * EST + c4);
        float x[4] = {a.x + bb.x, a.y + bb.y, a.z + bb.z, a.w + bb.w};
        if (resid_mode) {
          const float4 g = ga[i];
          float4 rr = rb[i];
          rr.x = fmaf(g.x, x[0], rr.x);
          rr.y = fmaf(g.y, x[1], rr.y);
          rr.z = fmaf(g.z, x[2], rr.z);
          rr.w = fmaf(g.w, x[3], rr.w);
          *reinterpret_cast<float4*>(e.resid + base) = rr;
          continue;
        }
        if (e.vec) {
          x[0] += ga[i].x; x[1] += ga[i].y; x[2] += ga[i].z; x[3] += ga[i].w;
        }
        if (e.resid) {
          x[0] += rb[i].x; x[1] += rb[i].y; x[2] += rb[i].z; x[3] += rb[i].w;
        }
        if (e.act)
#pragma unroll
          for (int j = 0; j < 4; ++j) x[j] = epi_gelu(e, x[j]);
        if (e.out)
          *reinterpret_cast<float4*>(e.out + base) = make_float4(x[0], x[1], x[2], x[3]);
        if (e.out_bf16) {
          __nv_bfloat162 p = __floats2bfloat162_rn(x[0], x[1]), q = __floats2bfloat162_rn(x[2], x[3]);
          uint2 u;
          u.x = *reinterpret_cast<uint32_t*>(&p);
          u.y = *reinterpret_cast<uint32_t*>(&q);
          *reinterpret_cast<uint2*>(e.out_bf16 + base) = u;
        }
      }
    }
    return;
  }
  auto row_pass = [&](int r0) {
    const int r = r0 + lane / LPR, grow = row0 + r;
    if (grow >= M || r >= nrows) return;
    for (int c4 = (lane % LPR) * 4; c4 < NC; c4 += LPR * 4) {
      if (col0 + c4 >= N) break;
      const float4 a = *reinterpret_cast<const float4*>(stg + r * EST + c4);
      const float v[4] = {a.x, a.y, a.z, a.w};
      epi_store4(e, grow, col0 + c4, N, v);
    }
  };
  // plain stores gain from 4 rows in flight (measured: 5% at CogVideoX
  // shapes); the GELU modes lose from it (register pressure)
  if (e.mode == EPI_STORE) {
#pragma unroll 4
    for (int r0 = 0; r0 < nrows; r0 += RPP) row_pass(r0);
  } else {
#pragma unroll 1
    for (int r0 = 0; r0 < nrows; r0 += RPP) row_pass(r0);
  }
}

// diagnostics (DIAG instantiation only): dbg bit 4 records clock64() phase
// stamps of CTA (0,0,0) here. Production launches use DIAG = false, so no
// diagnostic branch or clock read sits in the producer / MMA loops.
__device__ long long g_tc_ts[16];
#define TC_STAMP(i)                                                          \
  do {                                                                       \
    if (DIAG && (dbg & 16) && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) \
      g_tc_ts[i] = clock64();                                                \
  } while (0)

template <int KIND, int BN, bool DIAG>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapAlo,
                   const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapBlo,
                   int M, int N, int K, const __grid_constant__ Epi e, int dbg, TcSplit sk) {
  // dbg (diagnostics only, 0 in production): bit0 = no MMA, bit1 = no TMA
  using C = TcCfg<KIND, BN>;
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int TC_STAGES = C::STAGES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC_STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* accum = empty + TC_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * TC_BM, n0 = blockIdx.x * BN;
  if (!DIAG) dbg = 0;
  const int nk_all = (K + C::BK - 1) / C::BK;
  const int S = sk.splits;
  const int SC = sk.cluster;            // CTAs sharing the K range (1 = all in this CTA)
  const int G = S / SC;                 // consecutive segments per CTA
  const bool in_cta = SC == 1;
  const int zc = in_cta ? 0 : (int)blockIdx.z;
  const int kb0 = sk.seg[zc * G], kb1 = sk.seg[(zc + 1) * G];
  const int nk = kb1 - kb0;
  // TMEM columns: one BN-wide accumulator per segment of this CTA (power of 2 >= 32)
  uint32_t tcols = 32;
  while (tcols < (uint32_t)(G * BN)) tcols <<= 1;
  if (dbg & 8) return;  // probe: launch floor only
  if (threadIdx.x == 0) TC_STAMP(0);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    if (KIND == KIND_TF32X3) {
      tma_prefetch_desc(&mapAlo);
      tma_prefetch_desc(&mapBlo);
    }
    for (int s = 0; s < TC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TC_STAMP(1);
  // the prologue above overlaps the predecessor's tail (PDL); operands and
  // epilogue inputs are only touched after it completes - except the weight
  // tiles (B), which no kernel writes: the producer issues the first ring's
  // worth of B loads before its PDL wait, so their (HBM) latency overlaps the
  // predecessor's tail, then A once the predecessor is done
  const bool producer = warp == 0 && lane == 0;
  const int npre = (producer && !(dbg & 2)) ? (nk < TC_STAGES ? nk : TC_STAGES) : 0;
  for (int kb = 0; kb < npre; ++kb) {  // fresh ring: no empty waits
    uint8_t* st = smem + kb * C::STAGE_BYTES;
    mbar_expect_tx(&full[kb], C::STAGE_BYTES);
    const int kx = (kb0 + kb) * C::BK;
    tma_load_2d(st + C::A_BYTES, &mapB, &full[kb], kx, n0);
    if (KIND == KIND_TF32X3)
      tma_load_2d(st + 2 * C::A_BYTES + C::B_BYTES, &mapBlo, &full[kb], kx, n0);
  }
  pdl_wait_and_release();
  if (threadIdx.x == 0) TC_STAMP(2);

  if (producer) {
    // ---------------- TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % TC_STAGES;
      uint8_t* st = smem + s * C::STAGE_BYTES;
      const int kx = (kb0 + kb) * C::BK;
      if (kb < npre) {  // B already in flight: the A half of the stage
        tma_load_2d(st, &mapA, &full[s], kx, m0);
        if (KIND == KIND_TF32X3)
          tma_load_2d(st + C::A_BYTES + C::B_BYTES, &mapAlo, &full[s], kx, m0);
        continue;
      }
      mbar_wait(&empty[s], ((kb / TC_STAGES) & 1) ^ 1);
      if (dbg & 2) {
        mbar_expect_tx(&full[s], 0);
        continue;
      }
      mbar_expect_tx(&full[s], C::STAGE_BYTES);
      if (kb == 0) TC_STAMP(3);
      tma_load_2d(st, &mapA, &full[s], kx, m0);
      tma_load_2d(st + C::A_BYTES, &mapB, &full[s], kx, n0);
      if (KIND == KIND_TF32X3) {
        tma_load_2d(st + C::A_BYTES + C::B_BYTES, &mapAlo, &full[s], kx, m0);
        tma_load_2d(st + 2 * C::A_BYTES + C::B_BYTES, &mapBlo, &full[s], kx, n0);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp runs the loop (descriptor
    // arithmetic in uniform registers), one elected lane issues each op
    constexpr uint32_t idesc = make_idesc(KIND, TC_BM, BN);
    int seg = 0, seg_start = 0, seg_end = sk.seg[zc * G + 1] - kb0;
    for (int kb = 0; kb < nk; ++kb) {
      if (kb == seg_end) {  // next segment of this CTA: fresh accumulator columns
        ++seg;
        seg_start = kb;
        seg_end = sk.seg[zc * G + seg + 1] - kb0;
      }
      const uint32_t dacc = tmem + (uint32_t)(seg * BN);
      const int s = kb % TC_STAGES;
      mbar_wait(&full[s], (kb / TC_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (kb == 0) TC_STAMP(4);
      if (kb == nk - 1) TC_STAMP(5);
      uint8_t* st = smem + s * C::STAGE_BYTES;
      const uint64_t a0 = smem_desc_sw128(st);
      const uint64_t b0 = smem_desc_sw128(st + C::A_BYTES);
      if (dbg & 1) {
        mbar_arrive_e(&empty[s]);
        continue;
      }
#pragma unroll
      for (int k = 0; k < C::BK / C::UK; ++k) {
        // advance 32 B along K inside the swizzle atom: +2 in the >>4 address
        const uint64_t koff = (uint64_t)(k * C::UK * C::ESZ) >> 4;
        const uint32_t acc = ((kb - seg_start) | k) ? 1u : 0u;
        umma_e<KIND>(dacc, a0 + koff, b0 + koff, idesc, acc);
        if constexpr (KIND == KIND_TF32X3) {
          const uint64_t alo = smem_desc_sw128(st + C::A_BYTES + C::B_BYTES);
          const uint64_t blo = smem_desc_sw128(st + 2 * C::A_BYTES + C::B_BYTES);
          umma_e<KIND>(dacc, a0 + koff, blo + koff, idesc, 1u);
          umma_e<KIND>(dacc, alo + koff, b0 + koff, idesc, 1u);
        }
      }
      umma_commit_e(&empty[s]);
    }
    if (dbg & 1)
      mbar_arrive_e(accum);
    else
      umma_commit_e(accum);
  }
  __syncwarp();

  // ---------------- epilogue: TMEM -> registers -> fused store
  mbar_wait(accum, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) TC_STAMP(6);
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  if (in_cta) {
    // segments summed in order, staged per warp in the drained ring, then
    // written coalesced (warp_store_rows)
    constexpr int EST = BN + 4;
    float* stg = reinterpret_cast<float*>(smem) + warp * 32 * EST;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      tmem_ld16(trow + c, v);
      for (int sg = 1; sg < S; ++sg) {  // segment order 0..S-1
        float u[16];
        tmem_ld16(trow + sg * BN + c, u);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += u[j];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(stg + lane * EST + c + 4 * q) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    __syncwarp();
    if ((dbg & 4) == 0) warp_store_rows<BN, EST>(e, stg, m0 + warp * 32, n0, M, N, lane);
  } else {
    // this CTA's G segment partials -> own smem (the stage ring is drained:
    // all MMAs completed, every multicast into it has landed)
    constexpr int PST = BN + 4;  // row stride (floats), keeps 16-B alignment
    constexpr int PTILE = TC_BM * PST;
    float* part = reinterpret_cast<float*>(smem);
    const int rloc = warp * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < G * BN; c += 16) {  // segment c / BN -> partial tile c / BN
      float v[16];
      tmem_ld16(trow + c, v);
      float* dst = part + (c / BN) * PTILE + rloc * PST + (c % BN);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(dst + 4 * q) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    if (threadIdx.x == 0) TC_STAMP(9);
    cluster_sync_all();
    if (threadIdx.x == 0) TC_STAMP(10);
    // CTA z reduces rows [z*128/SC, (z+1)*128/SC) over DSMEM in segment order
    // seg_0 + seg_1 + ... (segment g lives in CTA g / G, partial g % G): the
    // same order as the in-CTA path, one float4 per thread per pass
    const int rows = TC_BM / SC, r0 = zc * rows;
    const int chunks = rows * (BN / 4);
    float* red = part + G * PTILE;  // this CTA's reduced rows [rows][PST], then the epilogue
    // gated residual / GELU: through the slab (coalesced rows, batched
    // residual loads); the other modes store straight from registers (the
    // slab measured slower for the U-Net's add / store epilogues)
    const bool slab = e.mode == EPI_RESID || e.mode == EPI_GELU;
    // SS segments: TC_REDUCE_LOADS / SS float4 chunks per thread per pass,
    // every remote load of a pass issued before the first use
    auto reduce = [&](auto seg_tag) {
      constexpr int SS = decltype(seg_tag)::value;
      constexpr int U = SS >= TC_REDUCE_LOADS ? 1 : TC_REDUCE_LOADS / SS;
      for (int base = threadIdx.x; base < chunks; base += U * TC_THREADS) {
        float4 a[U][SS];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * TC_THREADS;
          if (idx >= chunks) break;
          const int r = r0 + idx / (BN / 4), c = (idx % (BN / 4)) * 4;
          const float* src = part + r * PST + c;
#pragma unroll
          for (int sg = 0; sg < SS; ++sg)
            a[u][sg] = G == 1 ? ld_dsmem_f4(src, (uint32_t)sg)
                              : ld_dsmem_f4(src + (sg % G) * PTILE, (uint32_t)(sg / G));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * TC_THREADS;
          if (idx >= chunks) break;
          const int r = r0 + idx / (BN / 4), c = (idx % (BN / 4)) * 4;
          float4 v = a[u][0];
#pragma unroll
          for (int sg = 1; sg < SS; ++sg) {
            v.x += a[u][sg].x; v.y += a[u][sg].y; v.z += a[u][sg].z; v.w += a[u][sg].w;
          }
          if (slab) {
            *reinterpret_cast<float4*>(red + (r - r0) * PST + c) = v;
          } else if (m0 + r < M && n0 + c < N) {
            const float vv[4] = {v.x, v.y, v.z, v.w};
            epi_store4(e, m0 + r, n0 + c, N, vv);
          }
        }
      }
    };
    switch (S) {
      case 2: reduce(std::integral_constant<int, 2>{}); break;
      case 3: reduce(std::integral_constant<int, 3>{}); break;
      case 4: reduce(std::integral_constant<int, 4>{}); break;
      case 5: reduce(std::integral_constant<int, 5>{}); break;
      case 6: reduce(std::integral_constant<int, 6>{}); break;
      case 7: reduce(std::integral_constant<int, 7>{}); break;
      default: reduce(std::integral_constant<int, 8>{}); break;
    }
    if (slab) {  // coalesced epilogue over the reduced slab: rows / 4 rows per warp
      __syncthreads();
      const int rpw = rows / 4;
      if ((dbg & 4) == 0)
        warp_store_rows<BN, PST>(e, red + warp * rpw * PST, m0 + r0 + warp * rpw, n0, M, N, lane,
                                 rpw);
    }
    if (threadIdx.x == 0) TC_STAMP(11);
    cluster_sync_all();  // peers' smem stays live until every CTA has read it
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) TC_STAMP(7);
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(tcols));
  }
  if (threadIdx.x == 0) TC_STAMP(8);
}

// ------------------------------------------------------------------ 2-SM GEMM
// Large-M bf16 GEMM on CTA pairs (tcgen05 cta_group::2): one MMA instruction
// computes a 256 x 256 tile, A rows split across the pair (each CTA loads
// its own 128 rows) and B (the [N][K] weight copy) split likewise (each
// CTA loads 128 of the 256 N rows), so per CTA the operand traffic per
// output is half that of the 128 x 128 single-CTA tile - the large-M GEMMs
// are bound by L2 -> SM operand delivery, not by the tensor pipe.
//   both CTAs:  TMA of their A / B halves, signalling the LEADER's full
//               barrier (rank 0; the peer bit of the smem address cleared)
//   leader:     waits full, issues tcgen05.mma.cta_group::2 (M=256, N=256),
//               commits to BOTH CTAs' empty barriers (multicast), finally to
//               both CTAs' accumulator barriers
//   both CTAs:  epilogue from their own TMEM (128 rows x 256 columns)
// No split-K (S = 1): a row's accumulation order is the same K order as the
// single-CTA kernel.
constexpr int TC2_BN = 256, TC2_STAGES = 4;
constexpr int TC2_A_BYTES = 128 * 128, TC2_B_BYTES = 128 * 128;  // per CTA, per 64-K slab
constexpr int TC2_STAGE_BYTES = TC2_A_BYTES + TC2_B_BYTES;
constexpr int TC2_SMEM = TC2_STAGES * TC2_STAGE_BYTES + 1024 + 256;

static __global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    int M, int N, int K, const __grid_constant__ Epi e) {
  extern __shared__ __align__(1024) uint8_t tc2_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tc2_smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC2_STAGES * TC2_STAGE_BYTES);
  uint64_t* empty = full + TC2_STAGES;
  uint64_t* accum = empty + TC2_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int m0 = blockIdx.x * TC_BM;             // consecutive M tiles form the pair
  const int nb0 = blockIdx.y * TC2_BN;           // the pair's 256 N columns
  const int nh0 = nb0 + (int)rank * 128;         // this CTA's half of B
  const int nk = (K + 63) / 64;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    for (int s = 0; s < TC2_STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader only: its producer's arrive + both CTAs' bytes
      mbar_init(&empty[s], 1);  // one multicast commit from the leader's MMA
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TC2_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  cluster_sync_all();  // the leader's barriers exist before the peer's TMA signals them
  pdl_wait_and_release();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs), completion on the leader's barrier
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % TC2_STAGES;
      mbar_wait(&empty[s], ((kb / TC2_STAGES) & 1) ^ 1);
      const uint32_t bar = smem_u32(&full[s]) & 0xFEFFFFFFu;  // rank-0 CTA's barrier
      if (rank == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                     "r"(2 * TC2_STAGE_BYTES)
                     : "memory");
      uint8_t* st = smem + s * TC2_STAGE_BYTES;
      const int kx = kb * 64;
      asm volatile(
          "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(st)),
          "l"(reinterpret_cast<uint64_t>(&mapA)), "r"(bar), "r"(kx), "r"(m0)
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(st + TC2_A_BYTES)),
          "l"(reinterpret_cast<uint64_t>(&mapB)), "r"(bar), "r"(kx), "r"(nh0)
          : "memory");
    }
  } else if (warp == 1 && rank == 0) {
    // ---------------- MMA issuer (leader): M = 256 over the pair, N = 256;
    // whole warp in the loop, one elected lane issues
    constexpr uint32_t idesc = make_idesc(KIND_BF16, 256, TC2_BN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % TC2_STAGES;
      mbar_wait(&full[s], (kb / TC2_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint8_t* st = smem + s * TC2_STAGE_BYTES;
      const uint64_t a0 = smem_desc_sw128(st);
      const uint64_t b0 = smem_desc_sw128(st + TC2_A_BYTES);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t koff = (uint64_t)(k * 32) >> 4;
        const uint32_t acc = (kb | k) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(a0 + koff), "l"(b0 + koff), "r"(idesc), "r"(acc));
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
          " [%0], %1;\n\t}" ::"r"(smem_u32(&empty[s])),
          "h"((uint16_t)3)
          : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;\n\t}" ::"r"(smem_u32(accum)),
        "h"((uint16_t)3)
        : "memory");
  }
  __syncwarp();

  // ---------------- epilogue: this CTA's 128 rows x 256 columns from its
  // TMEM, 128 columns at a time staged per warp in the drained ring and
  // written coalesced (warp_store_rows)
  mbar_wait(accum, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  constexpr int EST = 128 + 4;
  float* stg = reinterpret_cast<float*>(smem) + warp * 32 * EST;
#pragma unroll 1
  for (int h = 0; h < TC2_BN; h += 128) {
#pragma unroll 1
    for (int c = 0; c < 128; c += 16) {
      float v[16];
      tmem_ld16(trow + h + c, v);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(stg + lane * EST + c + 4 * q) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    __syncwarp();
    warp_store_rows<128, EST>(e, stg, m0 + warp * 32, nb0 + h, M, N, lane);
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the peer's TMA / our commits are all done before either CTA exits
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TC2_BN));
  }
}

// ------------------------------------------------------------------ persistent 2-SM GEMM
// The 2-SM GEMM as a persistent kernel: one CTA pair per 2 SMs walks the
// pair tiles t = cluster, cluster + clusters, ... (N-tile fastest, so pairs
// running together share A rows in L2). TMEM holds two 256-column
// accumulators: while four epilogue warps drain tile i's accumulator
// (TMEM -> smem staging -> coalesced rows), the leader's MMA warp already
// accumulates tile i+1 into the other one - the epilogue, the prologue and
// the teardown leave the tensor pipe's critical path. Stage ring phases run
// on across tiles. Barriers: full/empty as in gemm_tc2_kernel; acc_full[b]
// (each CTA; the leader's multicast commit) and acc_empty[b] (the leader's;
// 8 arrivals = both CTAs' four epilogue warps, the peer's over DSMEM).
// Warps: 0 TMA, 1 MMA (leader), 2-5 epilogue (lane quarters 2, 3, 0, 1).
// Same MMA sequence per tile as gemm_tc2_kernel: bitwise-identical output.
constexpr int TC2P_STAGES = 4, TC2P_THREADS = 192;
constexpr int TC2P_EST = 128 + 4;
constexpr int TC2P_STG_BYTES = 4 * 32 * TC2P_EST * 4;  // per-warp epilogue staging
constexpr int TC2P_SMEM = TC2P_STAGES * TC2_STAGE_BYTES + TC2P_STG_BYTES + 1024 + 256;

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

static __global__ void __launch_bounds__(TC2P_THREADS, 1)
    gemm_tc2p_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, int M, int N, int K,
                     const __grid_constant__ Epi e) {
  extern __shared__ __align__(1024) uint8_t tc2p_smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tc2p_smem_raw) + 1023) & ~uintptr_t(1023));
  float* stg_all = reinterpret_cast<float*>(smem + TC2P_STAGES * TC2_STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC2P_STAGES * TC2_STAGE_BYTES +
                                               TC2P_STG_BYTES);
  uint64_t* empty = full + TC2P_STAGES;
  uint64_t* acc_full = empty + TC2P_STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;        // [2], leader's used
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int tiles_mp = (M + 255) / 256, tiles_n = (N + TC2_BN - 1) / TC2_BN;
  const int ntiles = tiles_mp * tiles_n;
  const int nk = (K + 63) / 64;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mapA);
    tma_prefetch_desc(&mapB);
    for (int s = 0; s < TC2P_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * TC2_BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  cluster_sync_all();  // the leader's barriers exist before the peer signals them
  pdl_wait_and_release();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs), completion on the leader's barrier
      int g = 0;
      for (int t = cl; t < ntiles; t += ncl) {
        const int m0 = (t / tiles_n) * 256 + (int)rank * 128;
        const int nh0 = (t % tiles_n) * TC2_BN + (int)rank * 128;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % TC2P_STAGES;
          mbar_wait(&empty[s], ((g / TC2P_STAGES) & 1) ^ 1);
          const uint32_t bar = smem_u32(&full[s]) & 0xFEFFFFFFu;  // rank-0 CTA's barrier
          if (rank == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                             smem_u32(&full[s])),
                         "r"(2 * TC2_STAGE_BYTES)
                         : "memory");
          uint8_t* st = smem + s * TC2_STAGE_BYTES;
          const int kx = kb * 64;
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::"
              "bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(st)),
              "l"(reinterpret_cast<uint64_t>(&mapA)), "r"(bar), "r"(kx), "r"(m0)
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::"
              "bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(st + TC2_A_BYTES)),
              "l"(reinterpret_cast<uint64_t>(&mapB)), "r"(bar), "r"(kx), "r"(nh0)
              : "memory");
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader), accumulator i & 1 for local tile i
      constexpr uint32_t idesc = make_idesc(KIND_BF16, 256, TC2_BN);
      int g = 0, i = 0;
      for (int t = cl; t < ntiles; t += ncl, ++i) {
        const int b = i & 1;
        mbar_wait_cluster(&acc_empty[b], ((i >> 1) & 1) ^ 1);  // both CTAs drained it
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dacc = tmem + (uint32_t)(b * TC2_BN);
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % TC2P_STAGES;
          mbar_wait(&full[s], (g / TC2P_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          uint8_t* st = smem + s * TC2_STAGE_BYTES;
          const uint64_t a0 = smem_desc_sw128(st);
          const uint64_t b0 = smem_desc_sw128(st + TC2_A_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t koff = (uint64_t)(k * 32) >> 4;
            const uint32_t acc = (kb | k) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dacc),
                "l"(a0 + koff), "l"(b0 + koff), "r"(idesc), "r"(acc));
          }
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::"
              "cluster.b64 [%0], %1;\n\t}" ::"r"(smem_u32(&empty[s])),
              "h"((uint16_t)3)
              : "memory");
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::"
            "cluster.b64 [%0], %1;\n\t}" ::"r"(smem_u32(&acc_full[b])),
            "h"((uint16_t)3)
            : "memory");
      }
    }
  } else {
    // ---------------- epilogue warps 2-5: TMEM lane quarter q = warp & 3
    const int q = warp & 3;
    float* stg = stg_all + q * 32 * TC2P_EST;
    int i = 0;
    for (int t = cl; t < ntiles; t += ncl, ++i) {
      const int b = i & 1;
      const int m0 = (t / tiles_n) * 256 + (int)rank * 128;
      const int nb0 = (t % tiles_n) * TC2_BN;
      mbar_wait(&acc_full[b], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t trow = tmem + (uint32_t)(b * TC2_BN) + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int h = 0; h < TC2_BN; h += 128) {
#pragma unroll 1
        for (int c = 0; c < 128; c += 16) {
          float v[16];
          tmem_ld16(trow + h + c, v);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<float4*>(stg + lane * TC2P_EST + c + 4 * j) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
        if (h + 128 >= TC2_BN) {  // accumulator b fully read: hand it back to the MMA
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(&acc_empty[b], 0u);
        }
        __syncwarp();
        warp_store_rows<128, TC2P_EST>(e, stg, m0 + q * 32, nb0 + h, M, N, lane);
        __syncwarp();
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // the peer's TMA / our commits / remote arrives are all done
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(2 * TC2_BN));
  }
}

// ------------------------------------------------------------------ host side
int tc_prepare(TcWeights& w, TcActs& acts, const std::vector<const float*>& Ws,
               const std::vector<int>& Ks, const std::vector<int>& Ns, int max_rows, int ref_rows,
               int D, int Dm, int precision);
// weights only; ref_rows[i] = one lane's rows of layer i (fixes its split-K)
int tc_prepare_weights(TcWeights& w, const std::vector<const float*>& Ws,
                       const std::vector<int>& Ks, const std::vector<int>& Ns,
                       const std::vector<int>& ref_rows, int precision);
int tc_gemm(const TcWeights& w, int layer, const TcOperand& A, int M, int N, int K, const Epi& e,
            int precision, cudaStream_t st);
void tc_release(TcWeights& w, TcActs& acts);
// 2-D K-major TMA map: dims {K, rows}, box {128 B of K, box_rows}, 128 B swizzle
int tc_make_map(CUtensorMap* m, const void* base, int esz, int K, int rows, int box_rows);
// the A operand's maps (op.rows x op.cols at op.bf16 / op.hi+op.lo), every multicast width
int tc_operand_maps(TcOperand& op, int precision);
// standalone test entry (C-ABI wrapper in gemm_tc.cu)
}  // namespace ps
