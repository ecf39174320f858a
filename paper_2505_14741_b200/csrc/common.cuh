// Shared device helpers: error plumbing, the counter RNG, the reverse step.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>
#include <utility>

#include "../../include/parastep_b200.h"

namespace ps {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

#define PS_TRY(expr)                                                         \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess)                                                   \
      return ::ps::fail((int)_e, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define PS_CHECK_ARG(cond, msg)                                              \
  do {                                                                       \
    if (!(cond)) return ::ps::fail(PS_EINVAL, msg);                          \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: every kernel of the denoise chain is
// launched with programmatic stream serialization, waits for its
// predecessor with griddepcontrol.wait before touching its outputs, and
// releases its own dependent right after (so at most two grids overlap:
// the next kernel's launch + prologue hides under this one's tail).
__device__ __forceinline__ void pdl_wait_and_release() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- RNG
// SplitMix64 finalizer and the (seed, stream) key: numerics.py:40-60.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed) ^ stream);
}

__host__ __device__ __forceinline__ uint64_t step_stream(int t) {
  return (1ull << 32) | (uint64_t)(uint32_t)t;  // (PURPOSE_STEP << 32) | t
}

// u = ((word >> 11) + 1) * 2^-53 in (0, 1]: numerics.py:63-66 (exact)
__device__ __forceinline__ double uniform_at(uint64_t key, uint64_t ctr) {
  uint64_t w = mix64(key ^ ctr);
  return __dmul_rn((double)((w >> 11) + 1ull), 1.1102230246251565e-16);
}

// Box-Muller pair at even counter b: numerics.py:69-80.
//   r = sqrt(-2 log u(b)), th = (2 pi) u(b+1); even -> r cos th, odd -> r sin th
__device__ __forceinline__ void normal_pair(uint64_t key, uint64_t b, double& n0, double& n1) {
  double u1 = uniform_at(key, b);
  double u2 = uniform_at(key, b + 1ull);
  double r = sqrt(__dmul_rn(-2.0, log(u1)));
  double th = __dmul_rn(6.283185307179586, u2);
  double s, c;
  sincos(th, &s, &c);
  n0 = __dmul_rn(r, c);
  n1 = __dmul_rn(r, s);
}

__device__ __forceinline__ double normal_at(uint64_t key, uint64_t ctr) {
  double a, b;
  normal_pair(key, ctr & ~1ull, a, b);
  return (ctr & 1ull) ? b : a;
}

// ---------------------------------------------------------------- reverse step
// schedule.py:111-114,125-131: m = (x - c*eps)/sqrt_a ; out = m + sigma*z
// (no FMA contraction: every op rounds like numpy float64)
__device__ __forceinline__ double ddpm(double x, double e, double c, double sa) {
  return __ddiv_rn(__dsub_rn(x, __dmul_rn(c, e)), sa);
}
__device__ __forceinline__ double ddpm_z(double x, double e, double c, double sa, double sig,
                                         double z) {
  return __dadd_rn(ddpm(x, e, c, sa), __dmul_rn(sig, z));
}

// ---------------------------------------------------------------- dtype io
template <typename T> struct Io;
template <> struct Io<double> {
  static __device__ __forceinline__ double ld(const double* p) { return *p; }
  static __device__ __forceinline__ void st(double* p, double v) { *p = v; }
};
template <> struct Io<float> {
  static __device__ __forceinline__ double ld(const float* p) { return (double)*p; }
  static __device__ __forceinline__ void st(float* p, double v) { *p = (float)v; }
};

}  // namespace ps
