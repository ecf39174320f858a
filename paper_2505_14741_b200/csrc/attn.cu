// Host side of the tcgen05 flash attention (attn_fmha.cuh) plus C-ABI
// diagnostics that run one attention against caller buffers.

#include <algorithm>
#include <cmath>
#include <mutex>

#include "attn_f32tc.cuh"
#include "attn_fmha.cuh"
#include "attn_mma.cuh"

namespace ps {

int fmha_make_map(CUtensorMap* m, const __nv_bfloat16* qkv_bf16, int rows, int cols) {
  return tc_make_map(m, qkv_bf16, 2, cols, rows, FM_BK);
}

template <int DH, int NQ, int POLY>
static cudaError_t fmha_go1(const CUtensorMap& map, const FmhaArgs& a, cudaStream_t st) {
  using C = FmCfg<DH, NQ>;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(fmha_tc_kernel<DH, NQ, POLY>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  });
  return launch_pdl(fmha_tc_kernel<DH, NQ, POLY>,
                    dim3((a.L + NQ * FM_BQ - 1) / (NQ * FM_BQ), a.H, a.B), dim3(C::THREADS),
                    C::SMEM, st, map, a);
}

static int g_fmha_nq = 0;     // test hook: force 1 or 2 query tiles per CTA (0 = auto)
static int g_fmha_poly = -1;  // test hook: exp pairs (of 4) on the polynomial (-1 = default)

// default share of polynomial exps per configuration (measured, profiles/)
template <int DH, int NQ>
constexpr int fmha_poly_default() { return DH == 64 ? 1 : 0; }  // same for NQ = 1 and 2: bits independent of the tiling

template <int DH, int NQ>
static cudaError_t fmha_go(const CUtensorMap& map, const FmhaArgs& a, cudaStream_t st) {
  const int poly = g_fmha_poly >= 0 ? g_fmha_poly : fmha_poly_default<DH, NQ>();
  return poly == 0 ? fmha_go1<DH, NQ, 0>(map, a, st)
                   : (poly == 1 ? fmha_go1<DH, NQ, 1>(map, a, st) : fmha_go1<DH, NQ, 2>(map, a, st));
}

int fmha_launch(const CUtensorMap& map, const FmhaArgs& a, cudaStream_t st) {
  const int DH = fmha_padded_dim(a.dh);
  if (DH == 0) return fail(PS_EUNSUP, "tcgen05 attention: head_dim must be a multiple of 8, <= 128");
  // two query tiles per CTA once the grid has enough CTAs for the SMs
  const int ctas1 = (a.L + FM_BQ - 1) / FM_BQ * a.H * a.B;
  const bool two = DH == 64 && (g_fmha_nq == 2 || (g_fmha_nq == 0 && ctas1 >= 4 * 148));
  cudaError_t e = DH == 128 ? fmha_go<128, 1>(map, a, st)
                            : (two ? fmha_go<64, 2>(map, a, st) : fmha_go<64, 1>(map, a, st));
  if (e != cudaSuccess) return fail((int)e, std::string("fmha: ") + cudaGetErrorString(e));
  return check_launch("fmha");
}

template <int NA, int KS>
static cudaError_t fmha_f32_go(const AttnArgs& a, int B, cudaStream_t st) {
  using C = F3Cfg<NA>;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(fmha_f32_kernel<NA, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::SMEM);
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.L + F3_BQ - 1) / F3_BQ * KS, a.H, B);
  cfg.blockDim = dim3(F3_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = KS;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fmha_f32_kernel<NA, KS>, a);
}

template <int NA>
static cudaError_t fmha_f32_ks(const AttnArgs& a, int B, cudaStream_t st) {
  // key blocks per query tile split over a cluster: 1, 2 or 4 CTAs
  const int nkb = (a.L + F3_BK - 1) / F3_BK;
  return nkb >= 4 ? fmha_f32_go<NA, 4>(a, B, st)
                  : (nkb >= 2 ? fmha_f32_go<NA, 2>(a, B, st) : fmha_f32_go<NA, 1>(a, B, st));
}

int fmha_f32_launch(const AttnArgs& a, int B, cudaStream_t st) {
  if (a.dh % 8 || a.dh > 64)
    return fail(PS_EUNSUP, "fp32 tcgen05 attention: head_dim must be a multiple of 8, <= 64");
  const cudaError_t e = a.dh <= 32 ? fmha_f32_ks<1>(a, B, st) : fmha_f32_ks<2>(a, B, st);
  if (e != cudaSuccess) return fail((int)e, std::string("fmha_f32: ") + cudaGetErrorString(e));
  return check_launch("fmha_f32");
}

static __global__ void f32_to_bf16_n(const float* in, __nv_bfloat16* out, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __float2bfloat16_rn(in[i]);
}

// fp32 [rows, 3, H, dh] -> bf16 [rows, 3, H, DH], zero-padded head dims
static __global__ void pad_qkv_bf16(const float* in, __nv_bfloat16* out, int64_t rows, int H,
                                    int dh, int DH) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)3 * H * DH;
  if (i >= rows * per) return;
  const int64_t r = i / per;
  const int j = (int)(i % per), wh = j / DH, d = j % DH;
  out[i] = d < dh ? __float2bfloat16_rn(in[r * 3 * H * dh + (int64_t)wh * dh + d])
                  : __float2bfloat16_rn(0.f);
}

static __global__ void bf16_to_f32_n(const __nv_bfloat16* in, float* out, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __bfloat162float(in[i]);
}

// One attention over qkv fp32 [B*L, 3D] (dh = D / H) into out fp32 [B*L, D]:
// impl 1 = mma.sync flash attention (bf16), impl 2 = tcgen05 FMHA (bf16,
// dh 64). `iters` > 0: return mean device us of that many back-to-back
// launches instead (qkv/out may then be null). Allocates; test/probe only.
static float attn_run(const float* qkv, float* out, int B, int L, int H, int D, int impl,
                      int iters, cudaStream_t st, int* rc_out) {
  const int dh = D / H, DH = fmha_padded_dim(dh);
  const int64_t nq = (int64_t)B * L * 3 * D, no = (int64_t)B * L * D;
  const int64_t nqp = (int64_t)B * L * 3 * H * (DH ? DH : 1);
  __nv_bfloat16 *qb = nullptr, *ob = nullptr;
  float *qf = nullptr, *out_f32 = nullptr;
  int rc = 0;
  float us = -1.f;
  if (cudaMalloc(&qb, std::max(nq, nqp) * 2) || cudaMalloc(&ob, no * 2) ||
      cudaMalloc(&qf, nq * 4) || cudaMalloc(&out_f32, no * 4)) {
    rc = fail(PS_ECUDA, "attn_run: cudaMalloc");
  }
  if (!rc) {
    if (qkv) {
      f32_to_bf16_n<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(qkv, qb, nq);
      // the mma.sync kernel reads fp32 qkv: give it the bf16-rounded values
      bf16_to_f32_n<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(qb, qf, nq);
      if (impl == 2 && DH)
        pad_qkv_bf16<<<(unsigned)((nqp + 255) / 256), 256, 0, st>>>(qf, qb, (int64_t)B * L, H, dh,
                                                                     DH);
    } else {
      cudaMemsetAsync(qb, 0, std::max(nq, nqp) * 2, st);
      cudaMemsetAsync(qf, 0, nq * 4, st);
    }
    CUtensorMap map;
    if (impl == 2) {
      if (!DH) rc = fail(PS_EUNSUP, "tcgen05 attention: unsupported head_dim");
      else rc = fmha_make_map(&map, qb, B * L, 3 * H * DH);
    }
    FmhaArgs fa{L, D, B, H, dh, 1.4426950408889634f / sqrtf((float)dh), ob};
    AttnArgs aa{};
    aa.qkv = qf;
    aa.L = L;
    aa.D = D;
    aa.H = H;
    aa.dh = dh;
    aa.scale = 1.0f / sqrtf((float)dh);
    aa.out_bf16 = ob;
    if (impl >= 5) aa.qkv = qkv ? qkv : qf;  // fp32 path reads the unrounded fp32 qkv
    if (impl >= 5) aa.out_bf16 = nullptr, aa.out_f32 = out_f32;
    auto go = [&]() -> int {
      if (impl == 2) return fmha_launch(map, fa, st);
      if (impl == 6) return fmha_f32_launch(aa, B, st);
      if (!launch_attn_tc(impl == 5 ? AM_TF32X3 : AM_BF16, aa, B, st))
        return fail(PS_EUNSUP, "head_dim unsupported");
      return check_launch("attn_tc");
    };
    if (!rc) rc = go();
    if (!rc && iters > 0) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
      for (int i = 0; i < iters && !rc; ++i) rc = go();
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      us = ms * 1000.f / iters;
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    if (!rc && out && impl >= 5)
      cudaMemcpyAsync(out, out_f32, no * 4, cudaMemcpyDeviceToDevice, st);
    else if (!rc && out)
      bf16_to_f32_n<<<(unsigned)((no + 255) / 256), 256, 0, st>>>(ob, out, no);
    cudaError_t se = cudaStreamSynchronize(st);
    if (!rc && se != cudaSuccess) rc = fail((int)se, std::string("attn: ") + cudaGetErrorString(se));
  }
  cudaFree(qb);
  cudaFree(ob);
  cudaFree(qf);
  cudaFree(out_f32);
  *rc_out = rc;
  return us;
}

}  // namespace ps

using namespace ps;

extern "C" {

int ps_attn_test(const float* qkv, float* out, int B, int L, int H, int D, int impl, void* cs) {
  PS_CHECK_ARG(qkv && out && B >= 1 && L >= 1 && H >= 1 && D % H == 0, "bad attention arguments");
  PS_CHECK_ARG(impl >= 1 && impl <= 6,
               "impl: 1 mma.sync bf16, 2 tcgen05 (auto), 3/4 tcgen05 1/2 tiles, 5 mma.sync 3xTF32, "
               "6 tcgen05 3xTF32");
  int rc = 0;
  g_fmha_nq = impl == 3 ? 1 : (impl == 4 ? 2 : 0);
  attn_run(qkv, out, B, L, H, D, impl >= 5 ? impl : (impl >= 2 ? 2 : 1), 0, as_stream(cs), &rc);
  g_fmha_nq = 0;
  return rc;
}

int ps_fmha_set_poly(int pairs) {
  PS_CHECK_ARG(pairs >= -1 && pairs <= 2, "pairs: -1 (default) or 0..2 of every 4");
  g_fmha_poly = pairs;
  return 0;
}

#ifdef FMHA_STAMPS
int ps_fmha_stamps(long long* out) {  // diagnostic build only
  return (int)cudaMemcpyFromSymbol(out, g_fm_ts, sizeof(g_fm_ts));
}
#endif

float ps_attn_probe(int B, int L, int H, int D, int impl, int iters) {
  if (B < 1 || L < 1 || H < 1 || D % H || iters < 1 || impl < 1 || impl > 6) return -1.f;
  int rc = 0;
  g_fmha_nq = impl == 3 ? 1 : (impl == 4 ? 2 : 0);
  float us = attn_run(nullptr, nullptr, B, L, H, D, impl >= 5 ? impl : (impl >= 2 ? 2 : 1), iters,
                      0, &rc);
  g_fmha_nq = 0;
  return rc ? -1.f : us;
}

}  // extern "C"
