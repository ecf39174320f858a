// Declarations of the tcgen05 flash attention (kernel in attn_fmha.cuh,
// host side in attn.cu), for callers that only launch it.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace ps {

// Q/K/V operand: bf16 [B*L, 3, H, DH] row-major (DH = fmha_padded_dim(dh):
// the head dim zero-padded to a whole number of 64-element swizzle atoms)
struct FmhaArgs {
  int L, D, B, H, dh;       // D = H * dh: the output row stride
  float scale_log2;         // log2(e) / sqrt(dh)
  __nv_bfloat16* out_bf16;  // [B*L, D], row-major (the proj GEMM's A operand)
};

// padded width for head_dim dh (dh % 8 == 0): 64 or 128; 0 = unsupported
inline int fmha_padded_dim(int dh) { return (dh % 8) ? 0 : (dh <= 64 ? 64 : (dh <= 128 ? 128 : 0)); }

// qkv_bf16: [rows, 3 * H * DH]; the map's box is 64 dims x 128 tokens
int fmha_make_map(CUtensorMap* m, const __nv_bfloat16* qkv_bf16, int rows, int cols);
int fmha_launch(const CUtensorMap& map, const FmhaArgs& a, cudaStream_t st);

// fp32 path (3xTF32 tcgen05, attn_f32tc.cuh): fp32 qkv [B*L, 3D] -> the
// proj GEMM's tf32 hi/lo (and/or fp32) operand; head_dim % 8 == 0, <= 64
struct AttnArgs;
int fmha_f32_launch(const AttnArgs& a, int B, cudaStream_t st);

}  // namespace ps
