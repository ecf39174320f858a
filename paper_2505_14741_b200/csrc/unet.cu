// U-Net-shaped noise predictor (BASELINE.json configs[4]): a native executor
// for the op list paper_2505_14741_b200/unet_spec.py plan() emits. The CPU
// oracle is oracle/unet.py.
//
// Activations are channels-last fp32 [B, H*W, C] (token-major: a 1x1 conv or
// a transformer linear is a plain GEMM over the same buffer). Every
// convolution is an implicit-GEMM on the bf16 tcgen05 kernel: one gather
// kernel writes the A operand [B*Ho*Wo, taps*Cin] in bf16 with GroupNorm
// (+SiLU), the skip concatenation, stride-2 / nearest-2x resampling and the
// zero padding fused in, and the GEMM epilogue adds bias, the ResBlock's
// time projection and the residual. Transformers reuse the DiT pieces
// (LN producer, tcgen05 attention, GELU epilogue).

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "attn_fmha.h"
#include "gemm_tc.cuh"

using namespace ps;

namespace ps {

enum { UOP_CONV = 0, UOP_LINEAR = 1, UOP_ATTN = 2 };
enum { PRE_NONE = 0, PRE_CONVERT = 1, PRE_GN = 2, PRE_GN_SILU = 3, PRE_LN = 4 };
enum { RS_NONE = 0, RS_DOWN = 1, RS_UP = 2 };
constexpr int BUF_LATENT = -2, BUF_EPS = -3;
constexpr int GN_MAX_SLICES = 32;

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ---------------------------------------------------------------- GroupNorm statistics
// stats[(b*G + g)*2 + {0,1}] = mean, rstd over the group's channels of the
// (virtual) concatenation [in1 | in2] and all pixels. Grid (G, B, S): block
// s takes a contiguous slice of the group's elements and writes its exact
// two-pass partial (count, mean, M2); the last block of the group to finish
// (atomic ticket) merges the S partials in slice order with Chan's formula.
// The result never depends on which block is last: deterministic.
struct GnArgs {
  const float* in1;
  const float* in2;
  int c1, c2, hw, G, S;
  float eps;
  float* partial;     // [B*G][S][3]
  unsigned* ticket;   // [B*G], zero between launches
  float* stats;
};

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.f;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) t += red[i];
  __syncthreads();
  return t;
}

static __global__ void __launch_bounds__(256) gn_stats_kernel(const __grid_constant__ GnArgs p) {
  __shared__ float red[32];
  __shared__ bool last;
  pdl_wait_and_release();
  const int g = blockIdx.x, b = blockIdx.y, sl = blockIdx.z;
  const int ctot = p.c1 + p.c2, cpg = ctot / p.G, cg0 = g * cpg;
  // slice = a contiguous pixel range; a thread walks pixels, reading the
  // group's cpg channels of each (contiguous: 16-byte loads when aligned and
  // inside one input of the concatenation); 32-bit index arithmetic
  const int px0 = (int)((int64_t)p.hw * sl / p.S), px1 = (int)((int64_t)p.hw * (sl + 1) / p.S);
  const bool one = cg0 + cpg <= p.c1 || cg0 >= p.c1;  // the group lies in in1 or in2
  const float* src = cg0 < p.c1 ? p.in1 : p.in2;
  const int cs = cg0 < p.c1 ? p.c1 : p.c2, co = cg0 < p.c1 ? cg0 : cg0 - p.c1;
  const bool vec = one && (cpg & 3) == 0 && (co & 3) == 0 && (cs & 3) == 0;
  const int rowb = b * p.hw;
  auto chan = [&](int row, int c) -> float {  // concatenated channel c of a row
    return c < p.c1 ? p.in1[(int64_t)row * p.c1 + c] : p.in2[(int64_t)row * p.c2 + (c - p.c1)];
  };
  auto pass = [&](float mean, bool sq) -> float {
    float acc = 0.f;
    for (int px = px0 + threadIdx.x; px < px1; px += blockDim.x) {
      const int row = rowb + px;
      if (vec) {
        const float4* q4 = reinterpret_cast<const float4*>(src + (int64_t)row * cs + co);
        for (int k = 0; k < (cpg >> 2); ++k) {
          const float4 v = q4[k];
          if (sq) {
            const float a = v.x - mean, c = v.y - mean, d = v.z - mean, e = v.w - mean;
            acc = fmaf(a, a, fmaf(c, c, fmaf(d, d, fmaf(e, e, acc))));
          } else {
            acc += (v.x + v.y) + (v.z + v.w);
          }
        }
      } else {
        for (int k = 0; k < cpg; ++k) {
          const float v = chan(row, cg0 + k);
          acc = sq ? fmaf(v - mean, v - mean, acc) : acc + v;
        }
      }
    }
    return acc;
  };
  const float cnt = (float)((px1 - px0) * cpg);
  const float mean = block_sum(pass(0.f, false), red) / cnt;
  const float m2 = block_sum(pass(mean, true), red);
  const int bg = b * p.G + g;
  if (threadIdx.x == 0) {
    float* pp = p.partial + ((int64_t)bg * p.S + sl) * 3;
    pp[0] = cnt;
    pp[1] = mean;
    pp[2] = m2;
    __threadfence();
    last = atomicAdd(&p.ticket[bg], 1u) == (unsigned)(p.S - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const volatile float* pp = p.partial + (int64_t)bg * p.S * 3;
    double na = pp[0], ma = pp[1], qa = pp[2];
    for (int k = 1; k < p.S; ++k) {  // Chan et al. pairwise merge, slice order
      const double nb = pp[3 * k], mb = pp[3 * k + 1], qb = pp[3 * k + 2];
      const double nn = na + nb, d = mb - ma;
      ma += d * nb / nn;
      qa += qb + d * d * na * nb / nn;
      na = nn;
    }
    p.stats[bg * 2] = (float)ma;
    p.stats[bg * 2 + 1] = rsqrtf((float)(qa / na) + p.eps);
    p.ticket[bg] = 0u;  // re-arm for the next launch / graph replay
  }
}

// ---------------------------------------------------------------- operand gather
// A[m, tap*Ctot + c] (bf16), m = b*Ho*Wo + oy*Wo + ox: one thread per
// (row, tap, 8-channel chunk), 16-byte stores along the row.
struct GatherArgs {
  const float* in1;
  const float* in2;
  int c1, c2, H, W, Ho, Wo, taps, resample, pre, in_chw, G;
  int64_t n_latent;  // in_chw: per-sample stride of the CHW latent
  const float* stats;
  __nv_bfloat16* A;
  int64_t total;  // rows * taps * chunks
};

static __global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ GatherArgs p) {
  pdl_wait_and_release();
  // 32-bit index arithmetic (the host keeps total < 2^31): 64-bit divisions
  // cost ~10x more per thread
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p.total) return;
  const int ctot = p.c1 + p.c2, chunks = ctot >> 3;
  const int mt = idx / chunks, chunk = idx - mt * chunks;
  const int m = mt / p.taps, tap = mt - m * p.taps;
  const int hwo = p.Ho * p.Wo;
  const int b = m / hwo, pix = m - b * hwo;
  const int oy = pix / p.Wo, ox = pix % p.Wo;
  int iy = oy, ix = ox;
  bool ok = true;
  if (p.taps == 9) {
    const int ky = tap / 3, kx = tap % 3;
    if (p.resample == RS_DOWN) {
      iy = 2 * oy - 1 + ky;
      ix = 2 * ox - 1 + kx;
    } else if (p.resample == RS_UP) {
      const int uy = oy - 1 + ky, ux = ox - 1 + kx;  // in the upsampled grid
      ok = uy >= 0 && uy < 2 * p.H && ux >= 0 && ux < 2 * p.W;
      iy = uy >> 1;
      ix = ux >> 1;
    } else {
      iy = oy - 1 + ky;
      ix = ox - 1 + kx;
    }
  }
  ok = ok && iy >= 0 && iy < p.H && ix >= 0 && ix < p.W;
  const int c0 = chunk * 8;
  float v[8];
  if (ok) {
    const int64_t srow = (int64_t)b * p.H * p.W + (int64_t)iy * p.W + ix;
    if (p.in_chw) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        v[k] = p.in1[(int64_t)b * p.n_latent + (int64_t)(c0 + k) * p.H * p.W +
                     (int64_t)iy * p.W + ix];
    } else {
      const float* src = c0 < p.c1 ? p.in1 + srow * p.c1 + c0 : p.in2 + srow * p.c2 + (c0 - p.c1);
      const float4 a = *reinterpret_cast<const float4*>(src);
      const float4 c = *reinterpret_cast<const float4*>(src + 4);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
    }
    if (p.pre == PRE_GN || p.pre == PRE_GN_SILU) {
      const int cpg = ctot / p.G;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int g = (c0 + k) / cpg;
        const float mean = p.stats[(b * p.G + g) * 2], rstd = p.stats[(b * p.G + g) * 2 + 1];
        float y = (v[k] - mean) * rstd;
        if (p.pre == PRE_GN_SILU) y = silu_f(y);
        v[k] = y;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 0.f;
  }
  uint4 u;
  u.x = pack_bf16x2(v[0], v[1]);
  u.y = pack_bf16x2(v[2], v[3]);
  u.z = pack_bf16x2(v[4], v[5]);
  u.w = pack_bf16x2(v[6], v[7]);
  *reinterpret_cast<uint4*>(p.A + (int64_t)m * (p.taps * ctot) + tap * ctot + c0) = u;
}

}  // namespace ps

struct UnetStep {
  ps_unet_op op;
  TcOperand A;        // the GEMM's A operand (scratch or a bf16 buffer) + its map
  CUtensorMap attn_map;
  int Ho, Wo, K;
};

struct ps_unet {
  ps_unet_config cfg;
  std::vector<UnetStep> steps;
  std::vector<void*> bufs;
  std::vector<const float*> W, b;
  const float* freq;
  int freq_rows;
  TcWeights tcw;
  std::vector<void*> owned;
  __nv_bfloat16* scratch = nullptr;  // im2col / producer output
  float* stats = nullptr;            // GroupNorm statistics
  float* gn_partial = nullptr;       // [B*G][GN_MAX_SLICES][3]
  unsigned* gn_ticket = nullptr;     // [B*G]
  float* zero_mod = nullptr;         // LN without modulation
  float *t1 = nullptr, *emb = nullptr, *temb = nullptr, *temb_b = nullptr;
  __nv_bfloat16* temb_w = nullptr;   // (temb_dim, temb_cols) bf16, all ResBlock projections
  int launches = 0;
};

static int ualloc(ps_unet* h, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) return fail((int)e, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  h->owned.push_back(*p);
  return 0;
}

static __global__ void f32_to_bf16_u(const float* in, __nv_bfloat16* out, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __float2bfloat16_rn(in[i]);
}

extern "C" {

int ps_unet_destroy(ps_unet* h) {
  if (!h) return 0;
  TcActs none;
  tc_release(h->tcw, none);
  for (void* p : h->owned) cudaFree(p);
  delete h;
  return 0;
}

int ps_unet_create(const ps_unet_config* cfg, const ps_dit_weights* w, ps_unet** out) {
  PS_CHECK_ARG(cfg && w && out && cfg->ops && cfg->bufs, "null argument");
  PS_CHECK_ARG(cfg->max_batch >= 1 && cfg->max_batch <= GV_MAXB, "max_batch must be in [1, 16]");
  PS_CHECK_ARG(cfg->groups >= 1 && cfg->groups <= 64, "groups must be in [1, 64]");
  ps_unet* h = new ps_unet();
  h->cfg = *cfg;
  h->bufs.assign(cfg->bufs, cfg->bufs + cfg->n_bufs);
  h->W.assign(w->W, w->W + w->n_layers);
  h->b.assign(w->b, w->b + w->n_layers);
  h->freq = w->freq_table;
  h->freq_rows = w->freq_rows;
  const int MB = cfg->max_batch, nl = w->n_layers;
  int rc = 0;
  auto bail = [&](int code) {
    ps_unet_destroy(h);
    return code;
  };
  // GEMM layers: the ops' weights go to the tensor cores (bf16, K-major copies)
  std::vector<const float*> Ws(nl, nullptr);
  std::vector<int> Ks(nl, 0), Ns(nl, 0), refs(nl, 1);
  size_t scratch = 0;
  for (int i = 0; i < cfg->n_ops; ++i) {
    const ps_unet_op& op = cfg->ops[i];
    UnetStep s{};
    s.op = op;
    s.Ho = op.resample == RS_DOWN ? op.h / 2 : (op.resample == RS_UP ? op.h * 2 : op.h);
    s.Wo = op.resample == RS_DOWN ? op.w / 2 : (op.resample == RS_UP ? op.w * 2 : op.w);
    const int ctot = op.c1 + op.c2;
    s.K = op.taps * ctot;
    if (op.kind != UOP_ATTN) {
      PS_CHECK_ARG(op.layer >= 0 && op.layer < nl, "op layer out of range");
      PS_CHECK_ARG(ctot % 8 == 0 && op.cout >= 1, "op channels must be multiples of 8");
      Ws[op.layer] = w->W[op.layer];
      Ks[op.layer] = s.K;
      Ns[op.layer] = op.cout;
      refs[op.layer] = s.Ho * s.Wo;
      if (op.pre != PRE_NONE) scratch = std::max(scratch, (size_t)MB * s.Ho * s.Wo * s.K);
    } else {
      PS_CHECK_ARG(op.heads * 64 == op.c1, "attention needs head_dim 64");
    }
    h->steps.push_back(s);
  }
  if ((rc = tc_prepare_weights(h->tcw, Ws, Ks, Ns, refs, 1))) return bail(rc);
  if ((rc = ualloc(h, (void**)&h->scratch, scratch * 2 + 256)) ||
      (rc = ualloc(h, (void**)&h->stats, (size_t)MB * cfg->groups * 2 * sizeof(float))) ||
      (rc = ualloc(h, (void**)&h->gn_partial,
                   (size_t)MB * cfg->groups * GN_MAX_SLICES * 3 * sizeof(float))) ||
      (rc = ualloc(h, (void**)&h->gn_ticket, (size_t)MB * cfg->groups * sizeof(unsigned))) ||
      (rc = ualloc(h, (void**)&h->zero_mod, 4096 * sizeof(float))) ||
      (rc = ualloc(h, (void**)&h->t1, (size_t)MB * cfg->temb_dim * sizeof(float))) ||
      (rc = ualloc(h, (void**)&h->emb, (size_t)MB * cfg->temb_dim * sizeof(float))) ||
      (rc = ualloc(h, (void**)&h->temb, (size_t)MB * cfg->temb_cols * sizeof(float) + 256)) ||
      (rc = ualloc(h, (void**)&h->temb_b, (size_t)cfg->temb_cols * sizeof(float) + 256)))
    return bail(rc);
  cudaMemset(h->zero_mod, 0, 4096 * sizeof(float));
  cudaMemset(h->gn_ticket, 0, (size_t)MB * cfg->groups * sizeof(unsigned));
  // concatenate every ResBlock's time projection into one (temb_dim, temb_cols) matrix
  {
    float* tw = nullptr;
    const size_t nw = (size_t)cfg->temb_dim * cfg->temb_cols;
    if ((rc = ualloc(h, (void**)&tw, nw * sizeof(float))) ||
        (rc = ualloc(h, (void**)&h->temb_w, nw * 2 + 256)))
      return bail(rc);
    for (const UnetStep& s : h->steps) {
      if (s.op.temb_layer < 0) continue;
      PS_CHECK_ARG(s.op.temb_off + s.op.cout <= cfg->temb_cols, "temb column out of range");
      cudaError_t e = cudaMemcpy2D(tw + s.op.temb_off, (size_t)cfg->temb_cols * sizeof(float),
                                   w->W[s.op.temb_layer], (size_t)s.op.cout * sizeof(float),
                                   (size_t)s.op.cout * sizeof(float), cfg->temb_dim,
                                   cudaMemcpyDeviceToDevice);
      if (e == cudaSuccess)
        e = cudaMemcpy(h->temb_b + s.op.temb_off, w->b[s.op.temb_layer], s.op.cout * sizeof(float),
                       cudaMemcpyDeviceToDevice);
      if (e != cudaSuccess) return bail(fail((int)e, "temb concat"));
    }
    f32_to_bf16_u<<<(unsigned)((nw + 255) / 256), 256>>>(tw, h->temb_w, nw);
  }
  // A-operand maps: the gather scratch, or the bf16 buffer a previous epilogue wrote
  for (UnetStep& s : h->steps) {
    const ps_unet_op& op = s.op;
    const int rows = MB * s.Ho * s.Wo;
    if (op.kind == UOP_ATTN) {
      PS_CHECK_ARG(op.in1 >= 0 && op.in1 < cfg->n_bufs && op.out >= 0, "attention buffers");
      if ((rc = fmha_make_map(&s.attn_map, (const __nv_bfloat16*)h->bufs[op.in1],
                              MB * op.h * op.w, 3 * op.c1)))
        return bail(rc);
      continue;
    }
    s.A.rows = rows;
    s.A.cols = s.K;
    s.A.bf16 = op.pre == PRE_NONE ? (__nv_bfloat16*)h->bufs[op.in1] : h->scratch;
    if ((rc = tc_operand_maps(s.A, 1))) return bail(rc);
  }
  gemv_set_attr<float>();
  gemv_set_attr<__nv_bfloat16>();
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(fail((int)e, std::string("unet create: ") + cudaGetErrorString(e)));
  *out = h;
  return 0;
}

int ps_unet_kernels_per_forward(const ps_unet* h) { return h ? h->launches : 0; }

int ps_unet_forward(ps_unet* h, const float* x, const int32_t* host_ts, int B, float* eps_out,
                    void* cs) {
  PS_CHECK_ARG(h && x && host_ts && eps_out, "null argument");
  PS_CHECK_ARG(B >= 1 && B <= h->cfg.max_batch, "batch exceeds max_batch");
  for (int b = 0; b < B; ++b)
    PS_CHECK_ARG(host_ts[b] >= 0 && host_ts[b] < h->freq_rows, "step index outside [0, T]");
  cudaStream_t st = as_stream(cs);
  const ps_unet_config& c = h->cfg;
  const int64_t n_latent = (int64_t)c.in_channels * c.height * c.width;
  int rc, launches = 0;
  // time conditioning: emb = SiLU(temb2(SiLU(temb1(freq[t])))), then every
  // ResBlock's projection of emb in one GEMV
  if ((rc = gemv(h->freq, c.freq_dim, host_ts, h->W[0], false, h->b[0], h->t1, c.freq_dim,
                 c.temb_dim, B, 1, st)))
    return rc;
  if ((rc = gemv(h->t1, c.temb_dim, nullptr, h->W[1], false, h->b[1], h->emb, c.temb_dim,
                 c.temb_dim, B, 1, st)))
    return rc;
  if ((rc = gemv(h->emb, c.temb_dim, nullptr, h->temb_w, true, h->temb_b, h->temb, c.temb_dim,
                 c.temb_cols, B, 0, st)))
    return rc;
  launches += 3;
  auto buf = [&](int id) -> float* { return id >= 0 ? (float*)h->bufs[id] : nullptr; };
  for (const UnetStep& s : h->steps) {
    const ps_unet_op& op = s.op;
    const int rows = B * s.Ho * s.Wo;
    if (op.kind == UOP_ATTN) {
      const FmhaArgs fa{op.h * op.w, op.c1, B, op.heads, 64, 1.4426950408889634f / 8.0f,
                        (__nv_bfloat16*)h->bufs[op.out]};
      if ((rc = fmha_launch(s.attn_map, fa, st))) return rc;
      ++launches;
      continue;
    }
    const float* in1 = op.in1 == BUF_LATENT ? x : buf(op.in1);
    // ---- A operand
    if (op.pre == PRE_GN || op.pre == PRE_GN_SILU) {
      // slices: ~2 blocks per SM for one lane, >= 1024 elements each; never a
      // function of B, so a lane's statistics are the same bits in any batch
      const int64_t n = (int64_t)op.h * op.w * ((op.c1 + op.c2) / c.groups);
      int S = (int)std::min<int64_t>(GN_MAX_SLICES, std::max<int64_t>(1, n / 1024));
      S = std::max(1, std::min(S, (2 * 148 + c.groups - 1) / c.groups));
      GnArgs g{in1, buf(op.in2), op.c1, op.c2, op.h * op.w, c.groups, S, op.eps,
               h->gn_partial, h->gn_ticket, h->stats};
      launch_pdl(gn_stats_kernel, dim3(c.groups, B, S), dim3(256), 0, st, g);
      if ((rc = check_launch("gn_stats"))) return rc;
      ++launches;
    }
    if (op.pre == PRE_LN) {
      LnModArgs p{};
      p.h = in1;
      p.rows = rows;
      p.D = op.c1;
      p.L = s.Ho * s.Wo;
      p.mod = h->zero_mod;
      p.mod_stride = 0;
      p.out_bf16 = h->scratch;
      const int threads = rows >= 148 * 16 ? 256 : 64;
      launch_pdl(ln_mod_kernel, dim3((rows * 32 + threads - 1) / threads), dim3(threads), 0, st, p);
      if ((rc = check_launch("ln"))) return rc;
      ++launches;
    } else if (op.pre != PRE_NONE) {
      GatherArgs g{};
      g.in1 = in1;
      g.in2 = buf(op.in2);
      g.c1 = op.c1;
      g.c2 = op.c2;
      g.H = op.h;
      g.W = op.w;
      g.Ho = s.Ho;
      g.Wo = s.Wo;
      g.taps = op.taps;
      g.resample = op.resample;
      g.pre = op.pre;
      g.in_chw = op.in1 == BUF_LATENT;
      g.G = c.groups;
      g.n_latent = n_latent;
      g.stats = h->stats;
      g.A = h->scratch;
      g.total = (int64_t)rows * op.taps * ((op.c1 + op.c2) / 8);
      PS_CHECK_ARG(g.total < (1ll << 31), "gather: operand too large for 32-bit indexing");
      launch_pdl(gather_kernel, dim3((unsigned)((g.total + 255) / 256)), dim3(256), 0, st, g);
      if ((rc = check_launch("gather"))) return rc;
      ++launches;
    }
    // ---- GEMM + fused epilogue
    Epi e{};
    e.bias = h->b[op.layer];
    if (op.out == BUF_EPS) {
      e.mode = EPI_NCHW;
      e.eps = eps_out;
      e.n_latent = n_latent;
      e.hw = s.Ho * s.Wo;
    } else {
      e.mode = EPI_ADD;
      e.L = s.Ho * s.Wo;
      if (op.temb_layer >= 0) {
        e.vec = h->temb + op.temb_off;
        e.vec_stride = c.temb_cols;
      }
      e.resid = buf(op.resid);
      if (op.out_bf16) e.out_bf16 = (__nv_bfloat16*)h->bufs[op.out];
      else e.out = buf(op.out);
      if (op.out2 >= 0) e.out_bf16 = (__nv_bfloat16*)h->bufs[op.out2];  // bf16 shadow
      e.act = op.act;
    }
    if ((rc = tc_gemm(h->tcw, op.layer, s.A, rows, op.cout, s.K, e, 1, st))) return rc;
    ++launches;
  }
  h->launches = launches;
  return 0;
}

}  // extern "C"
