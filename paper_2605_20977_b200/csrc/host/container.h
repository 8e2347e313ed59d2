// Sequence container (SPEC.md:555-559 BitstreamContainer; layout in
// FORMAT.md): a 64-byte little-endian header, then per frame the hyper and
// main payloads, each prefixed with its u32 length. The main payload is the
// multi-lane format (its lane table is the per-lane length
// header) or, for banded streams, the PSWB container of per-band payloads.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "pswa/pswa_cuda.h"

namespace pswa_host {

// Numerics revision of the device entropy model: 2 = SiLU via tanh.approx,
// softplus via __expf/__logf in the GEMM epilogues; 3 = the spatial blocks'
// down projections reduce K as two halves (split-K CTA pairs). A symbol
// decodes only under the exact mu/sigma that coded it, so streams of another
// numerics revision are refused instead of decoding to wrong latents.
constexpr uint16_t kContainerVersion = 3;
constexpr size_t kContainerHeader = 64;

struct ContainerHeader {
  uint32_t w_px = 0, h_px = 0, frames = 0, gop = 32, rate = 0, s = 4, N = 4;
  uint64_t cfg_hash = 0, weights_hash = 0;
  uint32_t prior = 0, n_bands = 1;
};

// Hash of everything the decoder must share with the encoder: the model
// architecture (canonical_cfg), the grid, the lane counts and the head family.
uint64_t stream_cfg_hash(const pswa_cfg& c, int n_bands);

void write_header(std::vector<uint8_t>& out, const ContainerHeader& h);
void append_frame(std::vector<uint8_t>& out, const uint8_t* hyper, size_t hl, const uint8_t* main,
                  size_t ml);

struct FrameRef {
  size_t hyper_off, hyper_len, main_off, main_len;
};
// Parses the header (throws HashError / invalid_argument on a bad header) and
// the frames present; a truncated tail frame is dropped (`complete` counts
// the whole frames available, <= header.frames).
ContainerHeader parse_container(const uint8_t* p, size_t len, std::vector<FrameRef>* frames);

}  // namespace pswa_host
