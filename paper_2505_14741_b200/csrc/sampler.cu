// The reuse-then-predict round on device: counter RNG, fused apply+roll.
//
// Reference semantics: numerics.py:56-120 (RNG), schedule.py:102-131
// (ddpm_step), engines.py:299-337 (cycle runner: roll lanes with their own
// cached eps, apply the fresh eps in round order).
//
// Layout: every sampler vector is a flat 1-D latent of n elements (fp64 or
// fp32), the same flatten order as the reference's numpy vector, so the RNG
// counter of element i is i. A thread owns VEC consecutive elements (16 B:
// 2 x fp64 or 4 x fp32) = 1 or 2 Box-Muller pairs, so both normals of a pair
// are produced by one log/sqrt/sincos. The per-element chain is kept in
// registers for the whole launch (apply steps, then each lane's roll; fp64
// for the fp64 state, fp32 for the DiT's fp32 state), so
// one launch reads x + c eps (+ lane caches) and writes x + lanes: the
// minimum traffic for the round.

#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace ps {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}
int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail((int)e, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

struct CycleParams {
  const void* x_in;
  void* x_out;
  int64_t n;
  const uint64_t* seed;
  int n_apply;
  int lane_lo, lane_hi;
  ps_step apply[PS_MAX_CYCLE];
  ps_step roll[PS_MAX_CYCLE];
  const void* eps[PS_MAX_CYCLE];
  void* rec[PS_MAX_CYCLE];
  const void* cache[PS_MAX_CYCLE];
  void* lane_out[PS_MAX_CYCLE];
  // fp32-state copies of apply/roll, rounded on the host (see cycle_f32_kernel)
  struct F32 {
    float c, inv_sa, sigma;
    int noisy;
  } fa[PS_MAX_CYCLE], fr[PS_MAX_CYCLE];
};

template <typename T, int VEC, bool SCALAR = false>
struct Vec {
  double v[VEC];
  __device__ __forceinline__ void load(const void* base, int64_t i0, int cnt) {
    const T* p = reinterpret_cast<const T*>(base) + i0;
    if (!SCALAR && cnt == VEC) {
      if constexpr (sizeof(T) == 4 && VEC == 4) {
        float4 f = *reinterpret_cast<const float4*>(p);
        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        return;
      } else if constexpr (sizeof(T) == 8 && VEC == 2) {
        double2 f = *reinterpret_cast<const double2*>(p);
        v[0] = f.x; v[1] = f.y;
        return;
      }
    }
#pragma unroll
    for (int k = 0; k < VEC; ++k) v[k] = (k < cnt) ? Io<T>::ld(p + k) : 0.0;
  }
  __device__ __forceinline__ void store(void* base, int64_t i0, int cnt) const {
    T* p = reinterpret_cast<T*>(base) + i0;
    if (!SCALAR && cnt == VEC) {
      if constexpr (sizeof(T) == 4 && VEC == 4) {
        *reinterpret_cast<float4*>(p) =
            make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
        return;
      } else if constexpr (sizeof(T) == 8 && VEC == 2) {
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
        return;
      }
    }
#pragma unroll
    for (int k = 0; k < VEC; ++k)
      if (k < cnt) Io<T>::st(p + k, v[k]);
  }
};

// z_t for VEC consecutive elements starting at even i0 (VEC even)
template <int VEC>
__device__ __forceinline__ void gen_z(uint64_t seed, int t, int64_t i0, double* z) {
  const uint64_t key = stream_key(seed, step_stream(t));
#pragma unroll
  for (int q = 0; q < VEC / 2; ++q) normal_pair(key, (uint64_t)(i0 + 2 * q), z[2 * q], z[2 * q + 1]);
}

template <typename T, int VEC, bool S>
__device__ __forceinline__ void step_vec(Vec<T, VEC, S>& x, const Vec<T, VEC, S>& e, const ps_step& s,
                                         const double* z) {
  if constexpr (sizeof(T) == 8) {
    // fp64 state: the reference's float64 arithmetic op for op (bit-exact)
#pragma unroll
    for (int k = 0; k < VEC; ++k)
      x.v[k] = s.noisy ? ddpm_z(x.v[k], e.v[k], s.c, s.sqrt_a, s.sigma, z[k])
                       : ddpm(x.v[k], e.v[k], s.c, s.sqrt_a);
  } else {
    // fp32 state: the same op order in IEEE fp32 (the fp32 path rounds every
    // stored state anyway; fp64 division would make the kernel FP64-bound)
    const float c = (float)s.c, sa = (float)s.sqrt_a, sg = (float)s.sigma;
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      float m = __fdiv_rn(__fsub_rn((float)x.v[k], __fmul_rn(c, (float)e.v[k])), sa);
      if (s.noisy) m = __fadd_rn(m, __fmul_rn(sg, (float)z[k]));
      x.v[k] = m;
    }
  }
}

constexpr int ZCACHE = 7;  // roll steps whose z stays in registers (degree <= 8)

template <typename T, int VEC, bool SCALAR>
__global__ void __launch_bounds__(256) cycle_kernel(const __grid_constant__ CycleParams p) {
  pdl_wait_and_release();
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC;
  if (i0 >= p.n) return;
  const int cnt = (p.n - i0) < VEC ? (int)(p.n - i0) : VEC;
  const uint64_t seed = *p.seed;

  Vec<T, VEC, SCALAR> x;
  x.load(p.x_in, i0, cnt);
  double z[VEC];
  // issue the first PF eps loads up front (independent 16 B loads in flight:
  // the kernel is HBM-bound at large n and latency-bound otherwise)
  constexpr int PF = 16 / VEC;  // 8 (fp64) / 4 (fp32) prefetched eps vectors
  Vec<T, VEC, SCALAR> ev[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k)
    if (k < p.n_apply) ev[k].load(p.eps[k], i0, cnt);
#pragma unroll
  for (int k = 0; k < PS_MAX_CYCLE; ++k) {
    if (k >= p.n_apply) break;
    const ps_step s = p.apply[k];
    if (p.rec[k]) x.store(p.rec[k], i0, cnt);
    Vec<T, VEC, SCALAR> e;
    if (k < PF) e = ev[k];
    else e.load(p.eps[k], i0, cnt);
    if (s.noisy) gen_z<VEC>(seed, s.t, i0, z);
    step_vec(x, e, s, z);
  }
  if (p.n_apply > 0) x.store(p.x_out, i0, cnt);

  if (p.lane_hi > 1) {
    const int nz = p.lane_hi - 1;  // lane j needs roll steps 0..j-1
    double zc[ZCACHE][VEC];
#pragma unroll
    for (int k = 0; k < ZCACHE; ++k)
      if (k < nz && p.roll[k].noisy) gen_z<VEC>(seed, p.roll[k].t, i0, zc[k]);
    for (int j = max(p.lane_lo, 1); j < p.lane_hi; ++j) {
      Vec<T, VEC, SCALAR> c, xj = x;
      c.load(p.cache[j], i0, cnt);
#pragma unroll
      for (int k = 0; k < ZCACHE; ++k)
        if (k < j) step_vec(xj, c, p.roll[k], zc[k]);
      for (int k = ZCACHE; k < j; ++k) {
        if (p.roll[k].noisy) gen_z<VEC>(seed, p.roll[k].t, i0, z);
        step_vec(xj, c, p.roll[k], z);
      }
      xj.store(p.lane_out[j], i0, cnt);
    }
  }
}

// ---------------------------------------------------------------------------
// fp32 state (the DiT predictors): the chain lives in fp32 registers, one
// float4 (16 B) per thread, and every eps vector of the round is loaded up
// front so 1 + c independent 16-B loads are in flight per thread (the kernel
// is a pure HBM stream at large n). The division by sqrt(alpha_t) becomes a
// multiplication by the host-rounded reciprocal: every op rounds explicitly
// (no contraction), so apply and roll chains are bit-identical wherever they
// compute the same step, and the fp32 path stays well inside its 1e-4 bound.
using F32Step = CycleParams::F32;

static F32Step f32_step_host(const ps_step& s) {
  return F32Step{(float)s.c, (float)(1.0 / s.sqrt_a), (float)s.sigma, s.noisy};
}

__device__ __forceinline__ float f32_ddpm(float x, float e, const F32Step& s, float z) {
  float m = __fmul_rn(__fsub_rn(x, __fmul_rn(s.c, e)), s.inv_sa);
  return s.noisy ? __fadd_rn(m, __fmul_rn(s.sigma, z)) : m;
}

template <bool AL>
__device__ __forceinline__ float4 f32_ld4(const void* base, int64_t i0, int cnt) {
  const float* p = reinterpret_cast<const float*>(base) + i0;
  if (AL && cnt == 4) return __ldg(reinterpret_cast<const float4*>(p));
  float v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = k < cnt ? __ldg(p + k) : 0.f;
  return make_float4(v[0], v[1], v[2], v[3]);
}

template <bool AL>
__device__ __forceinline__ void f32_st4(void* base, int64_t i0, int cnt, float4 v) {
  float* p = reinterpret_cast<float*>(base) + i0;
  if (AL && cnt == 4) {
    *reinterpret_cast<float4*>(p) = v;
    return;
  }
  const float a[4] = {v.x, v.y, v.z, v.w};
  for (int k = 0; k < cnt; ++k) p[k] = a[k];
}

__device__ __forceinline__ void f32_step4(float4& x, const float4& e, const F32Step& s,
                                          const float* z) {
  x.x = f32_ddpm(x.x, e.x, s, z[0]);
  x.y = f32_ddpm(x.y, e.y, s, z[1]);
  x.z = f32_ddpm(x.z, e.z, s, z[2]);
  x.w = f32_ddpm(x.w, e.w, s, z[3]);
}

__device__ __forceinline__ void f32_gen_z(uint64_t seed, const ps_step& s, int64_t i0, float* z) {
  if (!s.noisy) {
    z[0] = z[1] = z[2] = z[3] = 0.f;
    return;
  }
  double d[4];
  gen_z<4>(seed, s.t, i0, d);
#pragma unroll
  for (int k = 0; k < 4; ++k) z[k] = (float)d[k];
}

constexpr int F32_PF = 8;  // eps vectors loaded up front (c <= 8 covers degree <= 8)

// NOISY = some step of this launch adds sigma*z (posterior mode). In zero
// mode ("DDIM") no z is generated and the lane caches are loaded up front
// too; with z the per-lane caches are loaded one at a time instead, so the
// z registers of the roll steps fit.
template <bool AL, bool NOISY>
__global__ void __launch_bounds__(256, NOISY ? 2 : 4) cycle_f32_kernel(const __grid_constant__ CycleParams p) {
  pdl_wait_and_release();
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i0 >= p.n) return;
  const int cnt = (p.n - i0) < 4 ? (int)(p.n - i0) : 4;

  float4 x = f32_ld4<AL>(p.x_in, i0, cnt);
  float4 ev[F32_PF];
#pragma unroll
  for (int k = 0; k < F32_PF; ++k)
    if (k < p.n_apply) ev[k] = f32_ld4<AL>(p.eps[k], i0, cnt);
  float z[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < PS_MAX_CYCLE; ++k) {
    if (k >= p.n_apply) break;
    if (p.rec[k]) f32_st4<AL>(p.rec[k], i0, cnt, x);
    const float4 e = k < F32_PF ? ev[k] : f32_ld4<AL>(p.eps[k], i0, cnt);
    if (NOISY) f32_gen_z(*p.seed, p.apply[k], i0, z);
    f32_step4(x, e, p.fa[k], z);
  }
  if (p.n_apply > 0) f32_st4<AL>(p.x_out, i0, cnt, x);
  if (p.lane_hi <= 1) return;

  const int jlo = max(p.lane_lo, 1);
  if constexpr (!NOISY) {
    float4 cv[F32_PF];
#pragma unroll
    for (int j = 1; j < F32_PF; ++j)
      if (j >= jlo && j < p.lane_hi) cv[j] = f32_ld4<AL>(p.cache[j], i0, cnt);
#pragma unroll
    for (int j = 1; j < PS_MAX_CYCLE; ++j) {
      if (j >= p.lane_hi) break;
      if (j < jlo) continue;
      const float4 c = j < F32_PF ? cv[j] : f32_ld4<AL>(p.cache[j], i0, cnt);
      float4 xj = x;
      for (int k = 0; k < j; ++k) f32_step4(xj, c, p.fr[k], z);
      f32_st4<AL>(p.lane_out[j], i0, cnt, xj);
    }
  } else {
    const uint64_t seed = *p.seed;
    const int nz = p.lane_hi - 1;  // lane j needs roll steps 0..j-1
    float zc[ZCACHE][4];
#pragma unroll
    for (int k = 0; k < ZCACHE; ++k)
      if (k < nz) f32_gen_z(seed, p.roll[k], i0, zc[k]);
    for (int j = jlo; j < p.lane_hi; ++j) {
      const float4 c = f32_ld4<AL>(p.cache[j], i0, cnt);
      float4 xj = x;
#pragma unroll
      for (int k = 0; k < ZCACHE; ++k)
        if (k < j) f32_step4(xj, c, p.fr[k], zc[k]);
      for (int k = ZCACHE; k < j; ++k) {
        f32_gen_z(seed, p.roll[k], i0, z);
        f32_step4(xj, c, p.fr[k], z);
      }
      f32_st4<AL>(p.lane_out[j], i0, cnt, xj);
    }
  }
}

template <typename T>
__global__ void step_z_kernel(const T* x, const T* e, const T* z, T* out, int64_t n, ps_step s) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xv = Io<T>::ld(x + i), ev = Io<T>::ld(e + i);
  double r = s.noisy ? ddpm_z(xv, ev, s.c, s.sqrt_a, s.sigma, Io<T>::ld(z + i))
                     : ddpm(xv, ev, s.c, s.sqrt_a);
  Io<T>::st(out + i, r);
}

// one thread per Box-Muller pair
template <typename T>
__global__ void rng_normal_kernel(T* out, int64_t n, uint64_t key, uint64_t c0,
                                  const uint64_t* d_seed, uint64_t stream) {
  if (d_seed) key = stream_key(*d_seed, stream);  // graph-replayable seed
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // pair slot
  // element i = c0-relative; pair base counter b = (c0 + i) & ~1
  const uint64_t first_b = c0 & ~1ull;
  uint64_t b = first_b + 2ull * (uint64_t)j;
  int64_t i_even = (int64_t)(b - c0);  // may be -1 when c0 is odd
  if (i_even >= n) return;
  double a0, a1;
  normal_pair(key, b, a0, a1);
  if (i_even >= 0) Io<T>::st(out + i_even, a0);
  if (i_even + 1 < n) Io<T>::st(out + i_even + 1, a1);
}

template <typename T>
__global__ void rng_uniform_kernel(T* out, int64_t n, uint64_t key, uint64_t c0, double scale,
                                   int xavier) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double u = uniform_at(key, c0 + (uint64_t)i);
  // (2u - 1) * limit, rounded like numpy: predictor.py:211
  Io<T>::st(out + i, xavier ? __dmul_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0), scale) : u);
}

template <typename T>
static int launch_cycle(const CycleParams& p, cudaStream_t st, bool vec_ok) {
  constexpr int VEC = 16 / sizeof(T);
  cudaError_t e;
  if constexpr (sizeof(T) == 4) {
    // fp32 state: one float4 per thread (scalar accesses when unaligned)
    const int64_t threads = (p.n + 3) / 4;
    const int bs = threads >= 148 * 512 ? 256 : 64;
    const unsigned blocks = (unsigned)((threads + bs - 1) / bs);
    bool noisy = false;
    for (int k = 0; k < p.n_apply; ++k) noisy |= p.apply[k].noisy != 0;
    for (int k = 0; k + 1 < p.lane_hi; ++k) noisy |= p.roll[k].noisy != 0;
    const dim3 g(blocks), b(bs);
    if (vec_ok)
      e = noisy ? launch_pdl(cycle_f32_kernel<true, true>, g, b, 0, st, p)
                : launch_pdl(cycle_f32_kernel<true, false>, g, b, 0, st, p);
    else
      e = noisy ? launch_pdl(cycle_f32_kernel<false, true>, g, b, 0, st, p)
                : launch_pdl(cycle_f32_kernel<false, false>, g, b, 0, st, p);
    if (e != cudaSuccess) return fail((int)e, std::string("cycle_f32: ") + cudaGetErrorString(e));
    return check_launch("cycle_f32");
  } else {
  // small latents (e.g. 4096 elements): 64-thread blocks spread over more SMs
  if (vec_ok) {
    int64_t threads = (p.n + VEC - 1) / VEC;
    const int bs = threads >= 148 * 512 ? 256 : 64;
    unsigned blocks = (unsigned)((threads + bs - 1) / bs);
    e = launch_pdl(cycle_kernel<T, VEC, false>, dim3(blocks), dim3(bs), 0, st, p);
  } else {
    // unaligned buffers: 2 elements per thread, scalar loads
    int64_t threads = (p.n + 1) / 2;
    const int bs = threads >= 148 * 512 ? 256 : 64;
    unsigned blocks = (unsigned)((threads + bs - 1) / bs);
    e = launch_pdl(cycle_kernel<T, 2, true>, dim3(blocks), dim3(bs), 0, st, p);
  }
  if (e != cudaSuccess) return fail((int)e, std::string("cycle_kernel: ") + cudaGetErrorString(e));
  return check_launch("cycle_kernel");
  }
}

}  // namespace ps

using namespace ps;

extern "C" {

const char* ps_last_error(void) { return g_err.c_str(); }
int ps_version(void) { return 1; }

int ps_sm_count(int device) {
  int v = 0;
  PS_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  return v;
}

static int rng_normal(void* out, int64_t n, uint64_t seed, const uint64_t* d_seed,
                      uint64_t stream, uint64_t counter0, int dtype, void* cs) {
  PS_CHECK_ARG(n >= 1, "draw count must be >= 1");
  PS_CHECK_ARG(out != nullptr, "null output");
  uint64_t key = stream_key(seed, stream);
  int64_t pairs = (n + 2) / 2 + 1;
  unsigned blocks = (unsigned)((pairs + 255) / 256);
  if (dtype == PS_F64)
    rng_normal_kernel<double><<<blocks, 256, 0, as_stream(cs)>>>((double*)out, n, key, counter0,
                                                                  d_seed, stream);
  else if (dtype == PS_F32)
    rng_normal_kernel<float><<<blocks, 256, 0, as_stream(cs)>>>((float*)out, n, key, counter0,
                                                                 d_seed, stream);
  else
    return fail(PS_EUNSUP, "rng: dtype must be f64 or f32");
  return check_launch("rng_normal");
}

int ps_rng_normal(void* out, int64_t n, uint64_t seed, uint64_t stream, uint64_t counter0,
                  int dtype, void* cs) {
  return rng_normal(out, n, seed, nullptr, stream, counter0, dtype, cs);
}

int ps_rng_normal_dev(void* out, int64_t n, const uint64_t* d_seed, uint64_t stream,
                      uint64_t counter0, int dtype, void* cs) {
  PS_CHECK_ARG(d_seed != nullptr, "null seed pointer");
  return rng_normal(out, n, 0, d_seed, stream, counter0, dtype, cs);
}

static int rng_u(void* out, int64_t n, uint64_t seed, uint64_t stream, uint64_t c0, double scale,
                 int xavier, int dtype, void* cs) {
  PS_CHECK_ARG(n >= 1, "draw count must be >= 1");
  uint64_t key = stream_key(seed, stream);
  unsigned blocks = (unsigned)((n + 255) / 256);
  if (dtype == PS_F64)
    rng_uniform_kernel<double><<<blocks, 256, 0, as_stream(cs)>>>((double*)out, n, key, c0, scale,
                                                                   xavier);
  else if (dtype == PS_F32)
    rng_uniform_kernel<float><<<blocks, 256, 0, as_stream(cs)>>>((float*)out, n, key, c0, scale,
                                                                  xavier);
  else
    return fail(PS_EUNSUP, "rng: dtype must be f64 or f32");
  return check_launch("rng_uniform");
}

int ps_rng_uniform(void* out, int64_t n, uint64_t seed, uint64_t stream, uint64_t counter0,
                   int dtype, void* cs) {
  return rng_u(out, n, seed, stream, counter0, 1.0, 0, dtype, cs);
}

int ps_rng_xavier(void* out, int64_t n, uint64_t seed, uint64_t stream, double limit, int dtype,
                  void* cs) {
  return rng_u(out, n, seed, stream, 0, limit, 1, dtype, cs);
}

int ps_sched_cycle(const void* x_in, void* x_out, int64_t n, int dtype, const uint64_t* d_seed,
                   int n_apply, const ps_step* host_apply, const void* const* host_eps_apply,
                   void* const* host_rec_x, int lane_lo, int lane_hi, const ps_step* host_roll,
                   const void* const* host_lane_cache, void* const* host_lane_out, void* cs) {
  PS_CHECK_ARG(n >= 1, "vector length must be >= 1");
  PS_CHECK_ARG(d_seed != nullptr, "null seed pointer");
  PS_CHECK_ARG(n_apply >= 0 && n_apply <= PS_MAX_CYCLE, "n_apply out of range");
  PS_CHECK_ARG(lane_lo >= 0 && lane_hi <= PS_MAX_CYCLE && (lane_hi <= 1 || lane_lo < lane_hi),
               "lane range out of range");
  PS_CHECK_ARG(x_in != nullptr && (n_apply == 0 || x_out != nullptr), "null state pointer");
  CycleParams p;
  memset(&p, 0, sizeof(p));
  p.x_in = x_in;
  p.x_out = x_out;
  p.n = n;
  p.seed = d_seed;
  p.n_apply = n_apply;
  p.lane_lo = lane_lo;
  p.lane_hi = lane_hi;
  const size_t esz = dtype == PS_F64 ? 8 : 4;
  bool vec_ok = ((uintptr_t)x_in % 16 == 0) && ((uintptr_t)x_out % 16 == 0);
  for (int k = 0; k < n_apply; ++k) {
    p.apply[k] = host_apply[k];
    p.fa[k] = f32_step_host(host_apply[k]);
    p.eps[k] = host_eps_apply[k];
    PS_CHECK_ARG(p.eps[k] != nullptr, "null eps pointer");
    p.rec[k] = host_rec_x ? host_rec_x[k] : nullptr;
    vec_ok = vec_ok && ((uintptr_t)p.eps[k] % 16 == 0) && ((uintptr_t)p.rec[k] % 16 == 0);
  }
  if (lane_hi > 1) {
    for (int k = 0; k < lane_hi - 1; ++k) {
      p.roll[k] = host_roll[k];
      p.fr[k] = f32_step_host(host_roll[k]);
    }
    for (int j = (lane_lo > 1 ? lane_lo : 1); j < lane_hi; ++j) {
      p.cache[j] = host_lane_cache[j];
      p.lane_out[j] = host_lane_out[j];
      PS_CHECK_ARG(p.cache[j] != nullptr && p.lane_out[j] != nullptr, "null lane pointer");
      vec_ok = vec_ok && ((uintptr_t)p.cache[j] % 16 == 0) && ((uintptr_t)p.lane_out[j] % 16 == 0);
    }
  }
  (void)esz;
  if (dtype == PS_F64) return launch_cycle<double>(p, as_stream(cs), vec_ok);
  if (dtype == PS_F32) return launch_cycle<float>(p, as_stream(cs), vec_ok);
  return fail(PS_EUNSUP, "sched: dtype must be f64 or f32");
}

int ps_sched_step_z(const void* x, const void* eps, const void* z, void* out, int64_t n,
                    int dtype, const ps_step* s, void* cs) {
  PS_CHECK_ARG(n >= 1, "vector length must be >= 1");
  PS_CHECK_ARG(!s->noisy || z != nullptr, "noisy step needs z");
  unsigned blocks = (unsigned)((n + 255) / 256);
  if (dtype == PS_F64)
    step_z_kernel<double><<<blocks, 256, 0, as_stream(cs)>>>(
        (const double*)x, (const double*)eps, (const double*)z, (double*)out, n, *s);
  else if (dtype == PS_F32)
    step_z_kernel<float><<<blocks, 256, 0, as_stream(cs)>>>(
        (const float*)x, (const float*)eps, (const float*)z, (float*)out, n, *s);
  else
    return fail(PS_EUNSUP, "sched: dtype must be f64 or f32");
  return check_launch("step_z");
}

}  // extern "C"
