// Host side of the tcgen05 GEMM: operand preparation, TMA descriptors,
// launch; plus a C-ABI test entry that runs one GEMM against caller buffers.

#include <cstring>
#include <mutex>

#include "gemm_tc.cuh"

namespace ps {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encode() {
  if (g_encode) return 0;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000,
                                                   cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return fail(PS_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return 0;
}

// 2-D K-major map: dims {K, rows}, box {128 B of K, box_rows}, 128 B swizzle
int tc_make_map(CUtensorMap* m, const void* base, int esz, int K, int rows, int box_rows) {
  if (int rc = get_encode()) return rc;
  CUtensorMapDataType dt =
      esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * esz};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PS_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return 0;
}

// W (K, N) fp32 row-major -> Wt [N][K] as bf16, or as the tf32 hi/lo pair
__global__ void transpose_convert_kernel(const float* __restrict__ W, int K, int N,
                                         __nv_bfloat16* out_bf16, float* out_hi, float* out_lo) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int k = k0 + r, n = n0 + threadIdx.x;
    tile[r][threadIdx.x] = (k < K && n < N) ? W[(int64_t)k * N + n] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int n = n0 + r, k = k0 + threadIdx.x;
    if (n < N && k < K) {
      const float v = tile[threadIdx.x][r];
      const int64_t idx = (int64_t)n * K + k;
      if (out_bf16) out_bf16[idx] = __float2bfloat16_rn(v);
      if (out_hi) {
        const float hi = tf32_hi(v);
        out_hi[idx] = hi;
        out_lo[idx] = v - hi;
      }
    }
  }
}

int tc_operand_maps(TcOperand& op, int precision) {
  for (int i = 0; i < 1; ++i) {
    const int box = TC_BM;
    if (precision == 1) {
      if (int rc = tc_make_map(&op.map_main[i], op.bf16, 2, op.cols, op.rows, box)) return rc;
    } else {
      if (int rc = tc_make_map(&op.map_main[i], op.hi, 4, op.cols, op.rows, box)) return rc;
      if (int rc = tc_make_map(&op.map_lo[i], op.lo, 4, op.cols, op.rows, box)) return rc;
    }
  }
  return 0;
}

static int alloc_operand(TcActs& acts, TcOperand& op, int rows, int cols, int precision) {
  op.rows = rows;
  op.cols = cols;
  const size_t n = (size_t)rows * cols;
  cudaError_t e;
  if (precision == 1) {
    e = cudaMalloc(&op.bf16, n * 2);
    if (e != cudaSuccess) return fail((int)e, "cudaMalloc operand");
    acts.owned.push_back(op.bf16);
    cudaMemset(op.bf16, 0, n * 2);
    return tc_operand_maps(op, precision);
  }
  e = cudaMalloc(&op.hi, n * 4);
  if (e == cudaSuccess) {
    acts.owned.push_back(op.hi);
    e = cudaMalloc(&op.lo, n * 4);
  }
  if (e != cudaSuccess) return fail((int)e, "cudaMalloc operand");
  acts.owned.push_back(op.lo);
  cudaMemset(op.hi, 0, n * 4);
  cudaMemset(op.lo, 0, n * 4);
  return tc_operand_maps(op, precision);
}

static int cluster_cap(int s) { return s <= 2 ? 148 : 128; }  // co-resident CTAs

static int g_dbg = 0;  // ps_gemm_probe only
static int g_split_enable = 1;  // probe bit 5 disables split-K
static int g_force_in_cta = 0;  // probe bit 6 runs the segments in-CTA (no cluster)
static int g_sc_max = 8;        // test hook: cap on cluster CTAs along K (forces the hybrid)


static int bn_index(int bn) { return bn == 32 ? 0 : (bn == 64 ? 1 : 2); }

template <int KIND, int BN>
static int launch(const TcLayer& L, const TcOperand& A, int M, int N, int K, const Epi& e,
                  cudaStream_t st) {
  using C = TcCfg<KIND, BN>;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(gemm_tc_kernel<KIND, BN, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    cudaFuncSetAttribute(gemm_tc_kernel<KIND, BN, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  });
  const int tiles_n = (N + BN - 1) / BN, tiles_m = (M + TC_BM - 1) / TC_BM;
  // segments as a cluster only while the whole grid is co-resident (clusters
  // of 4/8 leave some SMs unusable, hence the lower cap); else in-CTA
  const int tiles = tiles_n * tiles_m;
  // K segments over as many cluster CTAs SC (| S) as stay co-resident, each
  // CTA running S/SC segments whose partial tiles fit its drained ring
  int sc = 1;
  if (!g_force_in_cta) {
    const size_t ring = (size_t)C::STAGES * C::STAGE_BYTES;
    const size_t ptile = (size_t)TC_BM * (BN + 4) * sizeof(float);
    for (int c = L.splits < g_sc_max ? L.splits : g_sc_max; c > 1; c /= 2) {
      // the CTA's partial tiles plus its reduced slab (128 / c rows) in the drained ring
      if (tiles * c <= cluster_cap(c) && (size_t)(L.splits / c) * ptile + ptile / c <= ring) {
        sc = c;
        break;
      }
    }
  }
  if ((L.splits / sc) * BN > 512)
    return fail(PS_EUNSUP, "gemm_tc: segment accumulators exceed the 512 TMEM columns");
  TcSplit sk{L.splits, sc, {}};
  const int nk_all = (K + C::BK - 1) / C::BK;
  for (int g = 0; g <= L.splits; ++g) sk.seg[g] = (int)((int64_t)g * nk_all / L.splits);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tiles_n, tiles_m, sk.cluster);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 1;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = sk.cluster;
  cfg.attrs = at;
  cfg.numAttrs = sk.cluster > 1 ? 2 : 1;
  const int bi = bn_index(BN);
  const CUtensorMap& alo = KIND == KIND_BF16 ? A.map_main[0] : A.map_lo[0];
  const CUtensorMap& blo = KIND == KIND_BF16 ? L.map_b[bi] : L.map_blo[bi];
  cudaError_t err = g_dbg ? cudaLaunchKernelEx(&cfg, gemm_tc_kernel<KIND, BN, true>, A.map_main[0],
                                               alo, L.map_b[bi], blo, M, N, K, e, g_dbg, sk)
                          : cudaLaunchKernelEx(&cfg, gemm_tc_kernel<KIND, BN, false>,
                                               A.map_main[0], alo, L.map_b[bi], blo, M, N, K, e, 0,
                                               sk);
  if (err != cudaSuccess) return fail((int)err, std::string("gemm_tc: ") + cudaGetErrorString(err));
  return check_launch("gemm_tc");
}

// 2-SM (cta_group::2) launch: 256 x 256 tiles on CTA pairs, bf16, no split.
static int g_force_2sm = -1;  // test hook: -1 auto, 0 never, 1 always (when legal)

static int launch2(const TcLayer& L, const TcOperand& A, int M, int N, int K, const Epi& e,
                   cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(gemm_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC2_SMEM);
  });
  const int tiles_m = (M + TC_BM - 1) / TC_BM;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((tiles_m + 1) / 2 * 2, (N + TC2_BN - 1) / TC2_BN, 1);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = TC2_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 2;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaError_t err =
      cudaLaunchKernelEx(&cfg, gemm_tc2_kernel, A.map_main[0], L.map_b[2], M, N, K, e);
  if (err != cudaSuccess) return fail((int)err, std::string("gemm_tc2: ") + cudaGetErrorString(err));
  return check_launch("gemm_tc2");
}

static int g_tc2_persistent = 1;  // test hook: 0 = one pair tile per CTA pair

// persistent 2-SM launch: one CTA pair per 2 SMs (at most 74 pairs), each
// walking pair tiles with a double-buffered TMEM accumulator
static int launch2p(const TcLayer& L, const TcOperand& A, int M, int N, int K, const Epi& e,
                    cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(gemm_tc2p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         TC2P_SMEM);
  });
  const int ntiles = ((M + 255) / 256) * ((N + TC2_BN - 1) / TC2_BN);
  const int pairs = std::min(ntiles, 74);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs, 1, 1);
  cfg.blockDim = dim3(TC2P_THREADS);
  cfg.dynamicSmemBytes = TC2P_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 2;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaError_t err =
      cudaLaunchKernelEx(&cfg, gemm_tc2p_kernel, A.map_main[0], L.map_b[2], M, N, K, e);
  if (err != cudaSuccess)
    return fail((int)err, std::string("gemm_tc2p: ") + cudaGetErrorString(err));
  return check_launch("gemm_tc2p");
}

// A layer takes the 2-SM kernel when one lane alone fills several waves of
// 128 x 128 tiles (decided from ref_rows, so every batch of the layer runs
// the same kernel: a row's bits never depend on the batch).
static bool use_2sm(const TcLayer& L, int precision) {
  if (precision != 1 || L.splits != 1 || g_force_2sm == 0) return false;
  if (g_force_2sm == 1) return true;
  // waves of 256 x 256 pair tiles (74 pairs per wave; one costs ~1.6 single-SM
  // 128 x 128 tile times, measured) against waves of 128 x 128 tiles
  const int tiles = ((L.ref_rows + TC_BM - 1) / TC_BM) * ((L.N + 127) / 128);
  const int pairs = ((L.ref_rows + 255) / 256) * ((L.N + TC2_BN - 1) / TC2_BN);
  const double w1 = (tiles + 147) / 148, w2 = (pairs + 73) / 74;
  return L.ref_rows >= 2048 && 1.6 * w2 < w1;
}

// Tile plan. At small M the mainloop is bound by per-SM TMA ingest
// (~70 GB/s/SM measured, profiles/): a CTA loads K/S x (128 + BN) operand
// elements, so wide N tiles (less re-reading of the shared A tile) plus
// split-K to fill the SMs beat narrow tiles. The planner scores every
// (BN, S) that fits co-resident (S <= 8 as one DSMEM cluster) by
//   ingest bytes per CTA + DSMEM reduction bytes (S > 1) + cluster-sync cost
// and keeps the cheapest. S is fixed per layer from the one-lane shape
// (ref_rows), so a row's accumulation order never depends on the batch
// (forward_batch == mapped forward, bitwise); BN may change per call.
static int g_split_min_kb = 2;  // ps_gemm_tune: K-blocks each split keeps at least (tf3x)
static int g_force_bn = 0, g_force_splits = 0;  // ps_gemm_force (calibration only)


struct TilePlan {
  int bn, splits;
};

static TilePlan plan_tiles_auto(int precision, int M, int N, int K);

// Measured overrides at the benchmarked batch-1 shapes (tools/gemm_plan_real.py:
// back-to-back launches of the real layers with every (BN, S) forced,
// profiles/r2_gemm_plan_real.txt); the cost model stays the fallback. A
// fixed table (not run-time autotuning) so every process and rank plans the
// same split-K order: bits never depend on timing noise.
struct PlanRule {
  int precision, M, N, K, bn, splits;
};
static const PlanRule kMeasuredPlans[] = {
    // DiT-S/2, 3xTF32 (auto: 7.32 / 6.27 / 8.55 / 7.96 us)
    {0, 256, 1152, 384, 32, 2},  // qkv 7.21
    {0, 256, 384, 384, 32, 4},   // proj 6.28
    {0, 256, 1536, 384, 32, 1},  // fc1 8.05
    {0, 256, 384, 1536, 64, 8},  // fc2 7.93
    // DiT-XL/2, bf16 (auto: 8.42 / 7.02 / 8.31 / 11.23 us)
    {1, 256, 3456, 1152, 32, 1},  // qkv 8.18
    {1, 256, 1152, 1152, 32, 1},  // proj 6.48
    {1, 256, 4608, 1152, 32, 1},  // fc1 8.03
    {1, 256, 1152, 4608, 32, 2},  // fc2 10.48
};

static TilePlan plan_tiles(int precision, int M, int N, int K) {
  TilePlan p = plan_tiles_auto(precision, M, N, K);
  for (const PlanRule& r : kMeasuredPlans)
    if (r.precision == precision && r.M == M && r.N == N && r.K == K) p = TilePlan{r.bn, r.splits};
  if (g_force_bn) p.bn = g_force_bn;
  if (g_force_splits) p.splits = g_force_splits;
  return p;
}

// Cost model fitted to the (BN, S) calibration grid (profiles/r1b_gemm_plan_grid.txt,
// tools/gemm_plan_grid.py), in microseconds per launch:
//   mainloop  = per-CTA operand ingest / 70 GB/s (per-SM TMA ingest)
//   split-K   = 1.3 (two cluster barriers) + the CTA's share of the DSMEM
//               reduction, 128 x BN x 4 B x (S-1)/S at ~25 GB/s
//   no split  = 0.3 (plain epilogue)
// (BN = 128, S = 8) measured far off the model (cluster placement) and is
// excluded. Grids beyond one wave pay per wave.
static TilePlan plan_tiles_auto(int precision, int M, int N, int K) {
  const int bk = precision == 1 ? 64 : 32;       // K elements per 128-byte stage row
  const double esz = precision == 1 ? 2.0 : 8.0;  // bytes per element incl. the tf32 lo copy
  const int nk = (K + bk - 1) / bk, tm = (M + TC_BM - 1) / TC_BM;
  TilePlan best{64, 1};
  double best_cost = 1e300;
  const int bns[3] = {32, 64, 128};
  for (int bn : bns) {
    const int tn = (N + bn - 1) / bn;
    for (int s = 1; s <= 8; s *= 2) {
      if (s > 1 && (tm * tn * s > cluster_cap(s) || nk / s < g_split_min_kb)) break;
      if (bn == 128 && s == 8) break;
      const int waves = (tm * tn * s + 147) / 148;
      double us = waves * ((double)((nk + s - 1) / s) * bk * (128 + bn) * esz / 70e3);
      us += s > 1 ? 1.3 + 128.0 * bn * 4 * (s - 1) / s / 25e3 : 0.3;
      if (us < best_cost * 0.98) {  // ties: the narrower / fewer-split plan
        best_cost = us;
        best = TilePlan{bn, s};
      }
    }
  }
  if (!g_split_enable) best.splits = 1;
  return best;
}

// N-tile width per call, for the layer's fixed split count: the planned
// width when the call is the planned shape, else narrow tiles for small
// grids and wide ones for large grids (in-CTA segments need S x BN <= 512
// TMEM columns). Any width gives the same per-element accumulation order.
static int choose_bn(const TcLayer& L, int precision, int M, int N) {
  const int splits = L.splits;
  const int tm = (M + TC_BM - 1) / TC_BM;
  auto fits = [&](int bn) {
    const int tiles = tm * ((N + bn - 1) / bn);
    return splits == 1 || tiles * splits <= cluster_cap(splits) || splits * bn <= 512;
  };
  if (M <= L.ref_rows && fits(L.bn)) return L.bn;
  const int t64 = tm * ((N + 63) / 64);
  if (2 * t64 * splits <= cluster_cap(splits)) return 32;
  if (t64 > 600 && splits * 128 <= 512) return 128;
  return 64;
}

int tc_prepare_weights(TcWeights& w, const std::vector<const float*>& Ws,
                       const std::vector<int>& Ks, const std::vector<int>& Ns,
                       const std::vector<int>& ref_rows, int precision) {
  w.precision = precision;
  w.layers.resize(Ws.size());
  for (size_t i = 0; i < Ws.size(); ++i) {
    TcLayer& L = w.layers[i];
    L.K = Ks[i];
    L.N = Ns[i];
    if (!Ws[i]) continue;  // placeholder (layer not run on the tensor cores)
    const TilePlan tp = plan_tiles(precision, ref_rows[i], L.N, L.K);
    L.splits = tp.splits;
    L.bn = tp.bn;
    L.ref_rows = ref_rows[i];
    const size_t n = (size_t)L.K * L.N;
    PS_CHECK_ARG(L.K % 8 == 0, "tensor-core GEMM needs K % 8 == 0");
    cudaError_t e;
    if (precision == 1) {
      e = cudaMalloc(&L.w_main, n * 2);
      if (e != cudaSuccess) return fail((int)e, "cudaMalloc weights");
    } else {
      e = cudaMalloc(&L.w_main, n * 4);
      if (e == cudaSuccess) e = cudaMalloc(&L.w_lo, n * 4);
      if (e != cudaSuccess) return fail((int)e, "cudaMalloc weights");
    }
    dim3 grid((L.N + 31) / 32, (L.K + 31) / 32), blk(32, 8);
    transpose_convert_kernel<<<grid, blk>>>(
        Ws[i], L.K, L.N, precision == 1 ? (__nv_bfloat16*)L.w_main : nullptr,
        precision == 1 ? nullptr : (float*)L.w_main, precision == 1 ? nullptr : (float*)L.w_lo);
    if (int rc = check_launch("transpose_convert")) return rc;
    const int boxes[3] = {32, 64, 128};
    for (int bi = 0; bi < 3; ++bi) {
      if (precision == 1) {
        if (int rc = tc_make_map(&L.map_b[bi], L.w_main, 2, L.K, L.N, boxes[bi])) return rc;
      } else {
        if (int rc = tc_make_map(&L.map_b[bi], L.w_main, 4, L.K, L.N, boxes[bi])) return rc;
        if (int rc = tc_make_map(&L.map_blo[bi], L.w_lo, 4, L.K, L.N, boxes[bi])) return rc;
      }
    }
  }
  return 0;
}

int tc_prepare(TcWeights& w, TcActs& acts, const std::vector<const float*>& Ws,
               const std::vector<int>& Ks, const std::vector<int>& Ns, int max_rows, int ref_rows,
               int D, int Dm, int precision) {
  const std::vector<int> refs(Ws.size(), ref_rows);
  if (int rc = tc_prepare_weights(w, Ws, Ks, Ns, refs, precision)) return rc;
  if (int rc = alloc_operand(acts, acts.a, max_rows, D, precision)) return rc;
  if (int rc = alloc_operand(acts, acts.o, max_rows, D, precision)) return rc;
  if (int rc = alloc_operand(acts, acts.hid, max_rows, Dm, precision)) return rc;
  return 0;
}

int tc_gemm(const TcWeights& w, int layer, const TcOperand& A, int M, int N, int K, const Epi& e,
            int precision, cudaStream_t st) {
  const TcLayer& L = w.layers[layer];
  if (use_2sm(L, precision))
    return g_tc2_persistent ? launch2p(L, A, M, N, K, e, st) : launch2(L, A, M, N, K, e, st);
  const int bn = choose_bn(L, precision, M, N);
  if (precision == 1) {
    if (bn == 32) return launch<KIND_BF16, 32>(L, A, M, N, K, e, st);
    if (bn == 128) return launch<KIND_BF16, 128>(L, A, M, N, K, e, st);
    return launch<KIND_BF16, 64>(L, A, M, N, K, e, st);
  }
  if (bn == 32) return launch<KIND_TF32X3, 32>(L, A, M, N, K, e, st);
  if (bn == 128) return launch<KIND_TF32X3, 128>(L, A, M, N, K, e, st);
  return launch<KIND_TF32X3, 64>(L, A, M, N, K, e, st);
}

void tc_release(TcWeights& w, TcActs& acts) {
  for (auto& L : w.layers) {
    if (L.w_main) cudaFree(L.w_main);
    if (L.w_lo) cudaFree(L.w_lo);
  }
  w.layers.clear();
  for (void* p : acts.owned) cudaFree(p);
  acts.owned.clear();
}

}  // namespace ps

using namespace ps;

namespace ps {
__global__ void convert_act_kernel(const float* src, __nv_bfloat16* bf, float* hi, float* lo,
                                   int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = src[i];
  if (bf) bf[i] = __float2bfloat16_rn(v);
  if (hi) {
    const float h = tf32_hi(v);
    hi[i] = h;
    lo[i] = v - h;
  }
}
}  // namespace ps

extern "C" {

// Test entry: C[M, N] = A[M, K] W[K, N] (+bias) on the tensor cores
// (precision 1 = bf16, 0 = 3xTF32) or the SIMT path (impl 1). A and W are
// fp32 device buffers in the reference layout; C fp32 [M, N]. Allocates and
// synchronises: test/diagnostic use only, never on the hot path.
int ps_gemm_test(const float* A, const float* W, const float* bias, float* Cout, int M, int N,
                 int K, int precision, int impl, void* cs) {
  PS_CHECK_ARG(M > 0 && N > 0 && K > 0, "bad GEMM shape");
  cudaStream_t st = as_stream(cs);
  // impl 3: tensor cores with the K segments forced in-CTA (cluster-free);
  // must equal impl 2 bit-for-bit (test_gemm_split_paths_bitwise)
  // impl 4: at most 2 cluster CTAs along K (each running S/2 segments);
  // impl 5 / 6: bf16 2-SM (cta_group::2) kernel forced on / off; 5 = one pair
  // tile per CTA pair, 7 = the persistent double-buffered 2-SM kernel
  g_force_in_cta = impl == 3 ? 1 : 0;
  g_sc_max = impl == 4 ? 2 : 8;
  g_force_2sm = (impl == 5 || impl == 7) ? 1 : (impl == 6 ? 0 : -1);
  g_tc2_persistent = impl == 5 ? 0 : 1;
  if (impl >= 3) impl = 2;
  Epi e{};
  e.mode = EPI_STORE;
  e.bias = bias;
  e.out = Cout;
  if (impl == 1) {
    dim3 grid((N + SG_BN - 1) / SG_BN, (M + SG_BM - 1) / SG_BM);
    gemm_simt_kernel<<<grid, 256, 0, st>>>(A, W, M, N, K, e);
    return check_launch("gemm_simt");
  }
  TcWeights w;
  TcActs acts;
  std::vector<const float*> Ws{W};
  std::vector<int> Ks{K}, Ns{N};
  int rc = tc_prepare(w, acts, Ws, Ks, Ns, M, M, K, K, precision);
  if (!rc) {
    const int64_t n = (int64_t)M * K;
    convert_act_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A, acts.a.bf16, acts.a.hi,
                                                                    acts.a.lo, n);
    rc = check_launch("convert_act");
  }
  if (!rc) rc = tc_gemm(w, 0, acts.a, M, N, K, e, precision, st);
  cudaError_t se = cudaStreamSynchronize(st);
  if (!rc && se != cudaSuccess) rc = fail((int)se, std::string("gemm_test: ") + cudaGetErrorString(se));
  tc_release(w, acts);
  g_force_in_cta = 0;
  g_sc_max = 8;
  g_force_2sm = -1;
  g_tc2_persistent = 1;
  return rc;
}


// Diagnostic: average device time (us) of `iters` back-to-back launches of
// the tensor-core GEMM on zero operands; dbg bit0 skips the MMAs, bit1 the
// TMA loads (pipeline-isolation experiments). Allocates; not hot path.
float ps_gemm_probe(int M, int N, int K, int precision, int dbg, int iters) {
  g_split_enable = (dbg & 32) ? 0 : 1;  // bit 5: disable split-K
  g_force_in_cta = (dbg & 64) ? 1 : 0;  // bit 6: segments in-CTA
  const bool resid_epi = (dbg & 1024) != 0;  // bit 10: gated-residual epilogue (EPI_RESID)
  const bool gelu_epi = (dbg & 4096) != 0;   // bit 12: GELU epilogue, next GEMM's operand format
  const bool nonzero = (dbg & 8192) != 0;    // bit 13: operands 0x3c3c3c3c (~0.0115), not 0
  g_force_2sm = (dbg & 2048) ? 0 : -1;       // bit 11: never the 2-SM kernel
  dbg &= 31;
  float *A = nullptr, *W = nullptr, *C = nullptr;
  if (cudaMalloc(&A, (size_t)M * K * 4) || cudaMalloc(&W, (size_t)K * N * 4) ||
      cudaMalloc(&C, (size_t)M * N * 4))
    return -1.f;
  cudaMemset(A, nonzero ? 0x3c : 0, (size_t)M * K * 4);
  cudaMemset(W, nonzero ? 0x3c : 0, (size_t)K * N * 4);
  float* C2 = nullptr;
  if (gelu_epi && cudaMalloc(&C2, (size_t)M * N * 4)) return -1.f;
  TcWeights w;
  TcActs acts;
  std::vector<const float*> Ws{W};
  std::vector<int> Ks{K}, Ns{N};
  float us = -1.f;
  if (!tc_prepare(w, acts, Ws, Ks, Ns, M, M, K, K, precision)) {
    Epi e{};
    e.mode = EPI_STORE;
    e.out = C;
    float* ones = nullptr;
    if (resid_epi) {
      cudaMalloc(&ones, (size_t)N * 4);
      cudaMemset(ones, 0, (size_t)N * 4);
      e.mode = EPI_RESID;
      e.resid = C;
      e.gate = ones;
      e.gate_stride = 0;
      e.L = M;
    }
    if (gelu_epi) {
      e.mode = EPI_GELU;
      e.out = nullptr;
      if (precision == 0) {
        e.out_hi = C;
        e.out_lo = C2;
      } else {
        e.out_bf16 = reinterpret_cast<__nv_bfloat16*>(C);
      }
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    g_dbg = dbg;
    tc_gemm(w, 0, acts.a, M, N, K, e, precision, 0);
    cudaEventRecord(a, 0);
    for (int i = 0; i < iters; ++i) tc_gemm(w, 0, acts.a, M, N, K, e, precision, 0);
    cudaEventRecord(b, 0);
    cudaEventSynchronize(b);
    g_dbg = 0;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    us = ms * 1000.f / iters;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (ones) cudaFree(ones);
  }
  cudaDeviceSynchronize();
  tc_release(w, acts);
  cudaFree(A);
  cudaFree(W);
  cudaFree(C);
  if (C2) cudaFree(C2);
  g_split_enable = 1;
  g_force_in_cta = 0;
  g_force_2sm = -1;
  return us;
}

// Tuning knob (diagnostic): minimum K-blocks per split-K segment; affects
// layers prepared afterwards. Returns the previous value.
// Calibration: force the planned (BN, S) of layers prepared afterwards
// (0 = planner's choice).
void ps_gemm_force(int bn, int splits) {
  g_force_bn = bn;
  g_force_splits = splits;
}

int ps_gemm_tune(int split_min_kb) {
  const int prev = g_split_min_kb;
  if (split_min_kb >= 1) g_split_min_kb = split_min_kb;
  return prev;
}

// Diagnostic: clock64 phase stamps of CTA (0,0,0) from the last probe run
// with dbg bit 4 set: [entry, prologue done, PDL wait done, first TMA
// issued, first stage landed (MMA), last stage landed, accumulator ready,
// epilogue done, exit].
int ps_gemm_stamps(long long* out12) {
  long long h[16];
  cudaError_t e = cudaMemcpyFromSymbol(h, g_tc_ts, sizeof(h));
  if (e != cudaSuccess) return fail((int)e, "stamps");
  for (int i = 0; i < 12; ++i) out12[i] = h[i];
  return 0;
}

}  // extern "C"
