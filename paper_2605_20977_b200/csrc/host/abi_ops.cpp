// Operator-level C-ABI entry points (device pointers): the per-op parity
// surface, mirroring the reference's per-op known-answer tests (SPEC.md:40-79,
// :221-256, :448-465).
#include <cuda_runtime.h>

#include <string>

#include "../cuda/check.h"
#include "../cuda/gemm.h"
#include "abi_util.h"
#include "pswa/pswa_cuda.h"

namespace pswa_abi {
namespace {
thread_local std::string g_last_error;
}
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace pswa_abi

extern "C" const char* pswa_gpu_last_error(void) { return pswa_abi::g_last_error.c_str(); }

extern "C" int pswa_gpu_op_gemm_f16(const void* A, int lda, int M, const void* B, int ldb, int N,
                                    int K, void* C, int ldc, int out_f32, int accumulate,
                                    const float* bias, const float* scale, int act, int force_bn,
                                    void* stream) {
  return pswa_abi::guard([&] {
    pswa_dev::GemmEpi ep;
    ep.out = C;
    ep.ld_out = ldc;
    ep.out_f32 = out_f32;
    ep.accumulate = accumulate;
    ep.bias = bias;
    ep.scale = scale;
    ep.act = act;
    if (act == pswa_dev::kActHead) ep.split = N / 2;
    pswa_dev::GemmPlan p;
    pswa_dev::gemm_plan(&p, static_cast<const __half*>(A), lda, M,
                        static_cast<const __half*>(B), ldb, N, K, ep, force_bn);
    pswa_dev::gemm_run(p, static_cast<cudaStream_t>(stream));
  });
}
