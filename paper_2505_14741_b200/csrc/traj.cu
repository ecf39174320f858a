// Trajectory diagnostics and serialisation on device.
//
// ps_traj_pack  writes the reference's binary trajectory file
//               (pkg/src/parastep/trajectory_io.py:100-110, "PSTJ" v1:
//               magic, <B version, <I steps, <I dim, then per record
//               <I t, <B fresh, x and eps as little-endian float64, then
//               x0) straight from the device tables, so a run's file is
//               one device pass + one D2H copy instead of T numpy records.
//               fp32 state widens exactly to float64.
// ps_traj_diff  per-row sums for compare_trajectories / rel_mae
//               (engines.py:446-473, numerics.py:144-158): sum|a-b|,
//               sum|a|, sum (a-b)^2 in fp64, one block per row with a
//               fixed-order reduction (deterministic).

#include <cstring>

#include "common.cuh"

namespace ps {

__device__ __forceinline__ double ld_state(const void* base, int dtype, int64_t i) {
  return dtype == PS_F64 ? reinterpret_cast<const double*>(base)[i]
                         : (double)reinterpret_cast<const float*>(base)[i];
}

__device__ __forceinline__ void st_bytes(uint8_t* dst, uint64_t bits, int nbytes) {
#pragma unroll
  for (int b = 0; b < 8; ++b)
    if (b < nbytes) dst[b] = (uint8_t)(bits >> (8 * b));  // little-endian
}

struct PackArgs {
  const void* rec_x;
  const void* eps;
  const void* x0;
  const int32_t* src_row;  // eps row consumed at record k
  const int32_t* ts;       // t of record k
  const uint8_t* fresh;
  int T, dtype;
  int64_t n;
  uint8_t* out;
};

static __global__ void traj_pack_kernel(const __grid_constant__ PackArgs p) {
  const int64_t rec_bytes = 5 + 16 * p.n;
  const int64_t vals = (int64_t)p.T * 2 * p.n + p.n;  // x, eps per record + x0
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    const uint8_t magic[4] = {'P', 'S', 'T', 'J'};
    for (int b = 0; b < 4; ++b) p.out[b] = magic[b];
    p.out[4] = 1;  // version
    st_bytes(p.out + 5, (uint32_t)p.T, 4);
    st_bytes(p.out + 9, (uint32_t)p.n, 4);
  }
  if (i < p.T) {  // record headers
    uint8_t* h = p.out + 13 + i * rec_bytes;
    st_bytes(h, (uint32_t)p.ts[i], 4);
    h[4] = p.fresh[i] ? 1 : 0;
  }
  if (i >= vals) return;
  double v;
  int64_t off;
  if (i < (int64_t)p.T * 2 * p.n) {
    const int64_t k = i / (2 * p.n), j = i % (2 * p.n);
    const bool is_x = j < p.n;
    const int64_t e = is_x ? j : j - p.n;
    v = is_x ? ld_state(p.rec_x, p.dtype, k * p.n + e)
             : ld_state(p.eps, p.dtype, (int64_t)p.src_row[k] * p.n + e);
    off = 13 + k * rec_bytes + 5 + 8 * j;
  } else {
    const int64_t e = i - (int64_t)p.T * 2 * p.n;
    v = ld_state(p.x0, p.dtype, e);
    off = 13 + (int64_t)p.T * rec_bytes + 8 * e;
  }
  st_bytes(p.out + off, (uint64_t)__double_as_longlong(v), 8);
}

struct DiffArgs {
  const void* a;
  const void* b;
  const int32_t* rows_a;  // optional row indirection (null = identity)
  const int32_t* rows_b;
  int dtype_a, dtype_b;
  int64_t n;
  double* out;  // [rows][3]
};

static __global__ void __launch_bounds__(256) traj_diff_kernel(const __grid_constant__ DiffArgs p) {
  __shared__ double red[3][8];
  const int r = blockIdx.x;
  const int64_t ra = p.rows_a ? p.rows_a[r] : r, rb = p.rows_b ? p.rows_b[r] : r;
  double sd = 0.0, sa = 0.0, sq = 0.0;
  for (int64_t i = threadIdx.x; i < p.n; i += blockDim.x) {
    const double x = ld_state(p.a, p.dtype_a, ra * p.n + i);
    const double y = ld_state(p.b, p.dtype_b, rb * p.n + i);
    const double d = x - y;
    sd += fabs(d);
    sa += fabs(x);
    sq = fma(d, d, sq);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sd += __shfl_xor_sync(0xffffffffu, sd, o);
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][w] = sd;
    red[1][w] = sa;
    red[2][w] = sq;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[threadIdx.x][k];
    p.out[r * 3 + threadIdx.x] = t;
  }
}

}  // namespace ps

using namespace ps;

extern "C" {

int64_t ps_traj_pack_bytes(int T, int64_t n) { return 13 + (int64_t)T * (5 + 16 * n) + 8 * n; }

int ps_traj_pack(const void* rec_x, const void* eps, const void* x0, const int32_t* src_row,
                 const int32_t* ts, const uint8_t* fresh, int T, int64_t n, int dtype, void* out,
                 void* cs) {
  PS_CHECK_ARG(rec_x && eps && x0 && src_row && ts && fresh && out, "null argument");
  PS_CHECK_ARG(T >= 0 && n >= 1, "bad trajectory shape");
  PS_CHECK_ARG(dtype == PS_F64 || dtype == PS_F32, "dtype must be f64 or f32");
  PackArgs p{rec_x, eps, x0, src_row, ts, fresh, T, dtype, n, (uint8_t*)out};
  const int64_t vals = (int64_t)T * 2 * n + n;
  const int64_t threads = vals > T ? vals : T;
  traj_pack_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(cs)>>>(p);
  return check_launch("traj_pack");
}

int ps_traj_diff(const void* a, const void* b, const int32_t* rows_a, const int32_t* rows_b,
                 int rows, int64_t n, int dtype_a, int dtype_b, double* out, void* cs) {
  PS_CHECK_ARG(a && b && out && rows >= 1 && n >= 1, "bad diff arguments");
  PS_CHECK_ARG((dtype_a == PS_F64 || dtype_a == PS_F32) && (dtype_b == PS_F64 || dtype_b == PS_F32),
               "dtype must be f64 or f32");
  DiffArgs p{a, b, rows_a, rows_b, dtype_a, dtype_b, n, out};
  traj_diff_kernel<<<rows, 256, 0, as_stream(cs)>>>(p);
  return check_launch("traj_diff");
}

}  // extern "C"
