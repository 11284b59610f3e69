// gemm.h — internal interface of the tcgen05 GEMM (csrc/gemm.cu).
#pragma once

#include <cuda_runtime.h>

#include "mrsp_c.h"

namespace mrsp {

struct GemmArgs {
  const void* A;  // [M][lda] bf16, K-major
  const void* B;  // [N][ldb] bf16, K-major (nn.Linear weight layout)
  void* C;        // output (bf16 or fp32 per epilogue)
  int M, N, K;
  int lda, ldb, ldc;
  int epi;              // mrsp_gemm_epilogue
  const float* bias;    // [N] fp32 or null
  float* resid;         // fp32 residual for GEMM_EPI_RESID_F32
  int ldr;
};

void gemm_bf16(const GemmArgs& g, cudaStream_t stream);

}  // namespace mrsp
