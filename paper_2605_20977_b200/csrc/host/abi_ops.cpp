// Operator-level C-ABI entry points (device pointers): the per-op parity
// surface, mirroring the reference's per-op known-answer tests (SPEC.md:40-79,
// :221-256, :448-465).
#include <cuda_runtime.h>

#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "../cuda/check.h"
#include "../cuda/gemm.h"
#include "../cuda/kernels.h"
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
    if (force_bn == -2) {  // split-K CTA pairs
      ep.split_k = 1;
      force_bn = 0;
    }
    pswa_dev::GemmPlan p;
    pswa_dev::gemm_plan(&p, static_cast<const __half*>(A), lda, M,
                        static_cast<const __half*>(B), ldb, N, K, ep, force_bn);
    pswa_dev::gemm_run(p, static_cast<cudaStream_t>(stream));
  });
}

// ---- the lane coder on explicit symbols -------------------
// Both run the production kernels: the encoder's lanes_encode + lanes_pack,
// and the decoder's lanes_init + decode_phase_kernel, driven as one phase of
// n single-channel positions whose (mu, sigma) = (0, scale[idx]) -- the
// phase decoder's sigma -> index rule then returns idx exactly (the 64 scales
// increase strictly).
namespace {
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { PSWA_CUDA(cudaMalloc(&p, bytes < 1 ? 1 : bytes)); }
  ~DevBuf() { cudaFree(p); }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

void check_idx(const int32_t* idx, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (idx[i] < 0 || idx[i] >= pswa_dev::kScales) throw std::invalid_argument("table index out of [0, 64)");
}
}  // namespace

extern "C" int pswa_gpu_op_encode_symbols(const int32_t* v, const int32_t* idx, size_t n, int lanes,
                                          int laplace, uint8_t* out, size_t cap, size_t* len,
                                          double* bits_out) {
  return pswa_abi::guard([&] {
    if (lanes < 1 || n > 0xFFFFFFFFull) throw std::invalid_argument("lanes < 1 or too many symbols");
    check_idx(idx, n);
    for (size_t i = 0; i < n; ++i)
      if (v[i] > INT32_MAX - 128 || v[i] < -(INT32_MAX - 128))
        throw std::invalid_argument("value outside the escape code's range");
    cudaStream_t st = nullptr;
    PSWA_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    DevBuf scales(sizeof(float) * pswa_dev::kScales), cdf(sizeof(uint32_t) * pswa_dev::kCdfWords);
    pswa_dev::build_cdf_tables(scales.as<float>(), cdf.as<uint32_t>(), st, laplace);
    std::vector<uint8_t> idx8(n);
    for (size_t i = 0; i < n; ++i) idx8[i] = static_cast<uint8_t>(idx[i]);
    DevBuf dv(sizeof(int32_t) * n), di(n);
    PSWA_CUDA(cudaMemcpyAsync(dv.p, v, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    PSWA_CUDA(cudaMemcpyAsync(di.p, idx8.data(), n, cudaMemcpyHostToDevice, st));
    const uint32_t lane_cap = static_cast<uint32_t>(16 * ((n + lanes - 1) / lanes) + 16);
    const uint64_t pcap = 12 + 4ull * lanes + static_cast<uint64_t>(lane_cap) * lanes;
    DevBuf enc(static_cast<size_t>(lane_cap) * lanes), lens(sizeof(uint32_t) * lanes),
        lbits(sizeof(double) * lanes), payload(pcap), total(2 * sizeof(unsigned long long)),
        offs(sizeof(uint64_t) * lanes), status(sizeof(int)), bits(sizeof(double));
    PSWA_CUDA(cudaMemsetAsync(status.p, 0, sizeof(int), st));
    pswa_dev::lanes_encode(dv.as<int32_t>(), di.as<uint8_t>(), n, lanes, cdf.as<uint32_t>(),
                           enc.as<uint8_t>(), lane_cap, lens.as<uint32_t>(), lbits.as<double>(),
                           status.as<int>(), st);
    pswa_dev::lanes_pack(enc.as<uint8_t>(), lane_cap, lens.as<uint32_t>(), lanes, static_cast<uint32_t>(n),
                         payload.as<uint8_t>(), pcap, total.as<unsigned long long>(), offs.as<uint64_t>(),
                         status.as<int>(), st);
    pswa_dev::sum_doubles(lbits.as<double>(), lanes, bits.as<double>(), st);
    unsigned long long tot = 0;
    int stat = 0;
    double b = 0;
    PSWA_CUDA(cudaMemcpyAsync(&tot, total.p, sizeof(tot), cudaMemcpyDeviceToHost, st));
    PSWA_CUDA(cudaMemcpyAsync(&stat, status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PSWA_CUDA(cudaMemcpyAsync(&b, bits.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    PSWA_CUDA(cudaStreamSynchronize(st));
    if (stat) throw pswa_abi::LaneError("encoder lane overrun (status " + std::to_string(stat) + ")");
    *len = tot;
    if (bits_out) *bits_out = b;
    if (out) {
      if (cap < tot) throw std::invalid_argument("output buffer too small");
      PSWA_CUDA(cudaMemcpy(out, payload.p, tot, cudaMemcpyDeviceToHost));
    }
  });
}

extern "C" int pswa_gpu_op_decode_symbols(const uint8_t* payload, size_t len, const int32_t* idx,
                                          size_t n, int laplace, int32_t* v_out, double* bits_out) {
  return pswa_abi::guard([&] {
    if (len < 12) throw pswa_abi::TruncatedError("payload shorter than its header");
    check_idx(idx, n);
    uint32_t L = 0;
    std::memcpy(&L, payload, 4);
    if (L < 1 || 12 + 2ull * L > len) throw pswa_abi::TruncatedError("bad lane count");
    cudaStream_t st = nullptr;
    PSWA_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    DevBuf scales(sizeof(float) * pswa_dev::kScales), cdf(sizeof(uint32_t) * pswa_dev::kCdfWords);
    pswa_dev::build_cdf_tables(scales.as<float>(), cdf.as<uint32_t>(), st, laplace);
    std::vector<float> sc(pswa_dev::kScales);
    PSWA_CUDA(cudaMemcpyAsync(sc.data(), scales.p, sizeof(float) * sc.size(), cudaMemcpyDeviceToHost, st));
    PSWA_CUDA(cudaStreamSynchronize(st));
    std::vector<float> musig(2 * n);
    std::vector<int> rows(n);
    for (size_t i = 0; i < n; ++i) {
      musig[2 * i] = 0.0f;
      musig[2 * i + 1] = sc[idx[i]];
      rows[i] = static_cast<int>(i);
    }
    // + 64 B: the phase decoder's byte reservoir reads up to 48 B past a lane
    DevBuf dp(len + 64), dlen(sizeof(uint32_t)), lanes(sizeof(pswa_dev::LaneState) * L),
        dms(sizeof(float) * 2 * n), drows(sizeof(int) * n), dy(sizeof(int32_t) * n),
        status(sizeof(int)), bits(sizeof(double));
    const uint32_t len32 = static_cast<uint32_t>(len);
    PSWA_CUDA(cudaMemsetAsync(dp.p, 0, len + 64, st));
    PSWA_CUDA(cudaMemcpyAsync(dp.p, payload, len, cudaMemcpyHostToDevice, st));
    PSWA_CUDA(cudaMemcpyAsync(dlen.p, &len32, sizeof(len32), cudaMemcpyHostToDevice, st));
    PSWA_CUDA(cudaMemcpyAsync(dms.p, musig.data(), sizeof(float) * 2 * n, cudaMemcpyHostToDevice, st));
    PSWA_CUDA(cudaMemcpyAsync(drows.p, rows.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
    PSWA_CUDA(cudaMemsetAsync(status.p, 0, sizeof(int), st));
    pswa_dev::lanes_init(dp.as<uint8_t>(), dlen.as<uint32_t>(), static_cast<int>(L), static_cast<uint32_t>(n),
                         lanes.as<pswa_dev::LaneState>(), status.as<int>(), st);
    // the phase decoder reads its lane states before its PDL wait (it relies
    // on a kernel between it and the lane init, as in the frame programs)
    PSWA_CUDA(cudaStreamSynchronize(st));
    pswa_dev::PhaseTaps taps;
    taps.ymax = INT32_MAX;
    pswa_dev::lanes_decode_phase(dp.as<uint8_t>(), lanes.as<pswa_dev::LaneState>(), static_cast<int>(L), 0,
                                 static_cast<int>(n), 1, dms.as<float>(), 2, 1, scales.as<float>(),
                                 cdf.as<uint32_t>(), drows.as<int>(), dy.as<int32_t>(), 1, 0, nullptr, 0,
                                 status.as<int>(), st, taps);
    pswa_dev::sum_lane_bits(lanes.as<pswa_dev::LaneState>(), static_cast<int>(L), bits.as<double>(), st);
    int stat = 0;
    double b = 0;
    PSWA_CUDA(cudaMemcpyAsync(&stat, status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PSWA_CUDA(cudaMemcpyAsync(&b, bits.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    if (n) PSWA_CUDA(cudaMemcpyAsync(v_out, dy.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    PSWA_CUDA(cudaStreamSynchronize(st));
    if (stat) throw pswa_abi::TruncatedError("corrupt or truncated lane payload (status " + std::to_string(stat) + ")");
    if (bits_out) *bits_out = b;
  });
}
