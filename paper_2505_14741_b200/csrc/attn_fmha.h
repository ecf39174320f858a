// Declarations of the tcgen05 flash attention (kernel in attn_fmha.cuh,
// host side in attn.cu), for callers that only launch it.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace ps {

struct FmhaArgs {
  int L, D, B;
  float scale_log2;         // log2(e) / sqrt(dh)
  __nv_bfloat16* out_bf16;  // [B*L, D], row-major (the proj GEMM's A operand)
};

constexpr int FM_HEAD_DIM = 64;  // the only head_dim the tcgen05 kernel takes

// qkv_bf16: [rows, 3D] row-major; the map's box is 64 dims x 128 tokens
int fmha_make_map(CUtensorMap* m, const __nv_bfloat16* qkv_bf16, int rows, int D);
int fmha_launch(const CUtensorMap& map, const FmhaArgs& a, int H, cudaStream_t st);

}  // namespace ps
