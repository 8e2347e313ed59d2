// Entropy coding on the device: quantised discretised-
// Gaussian CDF tables, and the multi-lane 64-bit-state range coder.
//
// Lane format (FORMAT.md §2): [u32 L][u32 count][u32 w][len_0..L-1, w bytes
// each: 2 when every lane is shorter than 64 KiB, else 4][lane 0 bytes]...;
// symbol ordinal o (canonical order: step, group, raster
// position, channel) lives in lane o % L. Each lane is an independent range
// coder with a 48-bit window (range in [2^40, 2^48)), big-endian byte
// renormalisation, carry into written bytes and a 4-byte flush; the decoder
// finds a symbol by multiply-compare binary search (no integer division).
// One thread drives one lane; lanes run concurrently, symbols within a lane
// sequentially.
//
// This file is compiled with -fmad=false: the fp64 table builder must round
// every add/mul exactly like the host restatement (det_math.cpp:49-130).
#include <cfloat>
#include <cstdint>

#include "check.h"
#include "kernels.h"
#include "launch.cuh"
#include "ptx.cuh"
#include "det_device.cuh"

namespace pswa_dev {

namespace {

constexpr uint64_t kWin = (uint64_t{1} << 48) - 1;
constexpr uint64_t kBot = uint64_t{1} << 40;
constexpr int kEscLo = 255, kEscHi = 256;
__device__ const uint32_t kBitCum[3] = {0, 32768, 65536};

__device__ __forceinline__ double sym_bits(uint32_t freq) {
  return 16.0 - log2(static_cast<double>(freq));
}

__host__ __device__ __forceinline__ uint16_t* sym_lut(uint32_t* cdf) {
  return reinterpret_cast<uint16_t*>(cdf + kScales * (kSyms + 1) + 2 * kScales * kSyms);
}
__host__ __device__ __forceinline__ const uint16_t* sym_lut(const uint32_t* cdf) {
  return reinterpret_cast<const uint16_t*>(cdf + kScales * (kSyms + 1) + 2 * kScales * kSyms);
}

__global__ void build_cdf_kernel(float* scales, uint32_t* cdf, int laplace) {
  pdl_wait();
  pdl_trigger();
  const int idx = threadIdx.x;
  if (idx >= kScales) return;
  const double ratio = d_log(64.0 / 0.11);
  const float sf = static_cast<float>(0.11 * d_exp(ratio * idx / 63.0));
  scales[idx] = sf;
  const double sigma = sf;
  const double inv = 1.0 / (sigma * 1.4142135623730951);
  uint32_t freq[kSyms];
  auto q = [](double p) -> uint32_t {
    if (p < 0.0) p = 0.0;
    return 1u + static_cast<uint32_t>(floor(p * 65279.0));
  };
  if (!laplace) {  // Gaussian: p(v) = Phi((v+1/2)/sigma) - Phi((v-1/2)/sigma)
    freq[127] = q(d_erf(0.5 * inv));
    for (int v = 1; v <= 127; ++v) {
      const double p = 0.5 * (d_erf((v + 0.5) * inv) - d_erf((v - 0.5) * inv));
      freq[127 + v] = freq[127 - v] = q(p);
    }
    freq[kEscLo] = freq[kEscHi] = q(0.5 * (1.0 - d_erf(127.5 * inv)));
  } else {  // Laplace, scale b = sigma: F(x) = 1 - exp(-x/b) / 2 for x >= 0
    const double ib = 1.0 / sigma;
    freq[127] = q(1.0 - d_exp(-0.5 * ib));
    for (int v = 1; v <= 127; ++v) {
      const double p = 0.5 * (d_exp(-(v - 0.5) * ib) - d_exp(-(v + 0.5) * ib));
      freq[127 + v] = freq[127 - v] = q(p);
    }
    freq[kEscLo] = freq[kEscHi] = q(0.5 * d_exp(-127.5 * ib));
  }
  uint32_t sum = 0;
  for (int k = 0; k < kSyms; ++k) sum += freq[k];
  freq[127] += 65536u - sum;
  uint32_t* c = cdf + idx * (kSyms + 1);
  c[0] = 0;
  for (int k = 0; k < kSyms; ++k) c[k + 1] = c[k] + freq[k];
  double* bt = reinterpret_cast<double*>(cdf + kScales * (kSyms + 1)) + idx * kSyms;
  for (int k = 0; k < kSyms; ++k) bt[k] = sym_bits(freq[k]);
  uint16_t* lut = sym_lut(cdf) + idx * kLutBuckets;
  int k = 0;
  for (int b = 0; b < kLutBuckets; ++b) {  // largest k < kSyms with c[k] <= b * 256
    while (k + 1 < kSyms && c[k + 1] <= static_cast<uint32_t>(b) * 256u) ++k;
    lut[b] = static_cast<uint16_t>(k);
  }
  // bit 15 of entry b: every symbol strictly between lut[b] and lut[b + 1]
  // has frequency 1 (the distribution's tails), so the decoder finds the
  // symbol of a target in bucket b in closed form instead of searching
  for (int b = 0; b + 1 < kLutBuckets; ++b) {
    bool unit = true;
    for (int j = lut[b] + 1; j < (lut[b + 1] & 0x7fff); ++j) unit = unit && freq[j] == 1u;
    if (unit) lut[b] |= 0x8000u;
  }
}

// ------------------------------------------------------------ helpers -----
// Smallest i with scales[i] >= sigma (63 when none, NaN included): a log2
// estimate of i (the scales are log-spaced, 0.146 octaves apart) corrected
// against the table itself, so the result is exactly the binary search's
// (the correction loops run 0-1 steps) with 2 dependent table reads instead
// of 6.
__device__ __forceinline__ int scale_index(const float* scales, float sigma) {
  if (!(sigma <= scales[kScales - 1])) return kScales - 1;
  constexpr float kLog2Lo = -3.184424571f;                  // log2(0.11)
  constexpr float kPerOctave = 63.0f / 9.184424571f;        // 63 / log2(64 / 0.11)
  int i = __float2int_ru((__log2f(sigma) - kLog2Lo) * kPerOctave);
  i = min(max(i, 0), kScales - 1);
  while (i > 0 && scales[i - 1] >= sigma) --i;
  while (i < kScales - 1 && scales[i] < sigma) ++i;
  return i;
}

__device__ __forceinline__ uint32_t rd32(const uint8_t* p) {
  return p[0] | (p[1] << 8) | (p[2] << 16) | (static_cast<uint32_t>(p[3]) << 24);
}

__device__ __forceinline__ uint32_t next_byte(const uint8_t* pl, LaneState& s, int& err) {
  if (s.pos < s.end) return pl[s.pos++];
  if (s.pos < s.end + 2) {
    ++s.pos;
    return 0;
  }
  err = 1;
  return 0;
}

// Payload byte reader: one global load per byte (the hyperprior lanes; the
// phase decoder uses the Rsv reservoir below).
struct ByteDirect {
  const uint8_t* pl;
  __device__ __forceinline__ uint32_t get(LaneState& s, int& err) { return next_byte(pl, s, err); }
};

template <class R>
__device__ __forceinline__ int dec_sym(R& rd, LaneState& s, const uint32_t* cum, int nsym, int& err) {
  const uint64_t r = s.range >> 16;
  if (s.code >= (r << 16)) {
    err = 1;
    s.code = (r << 16) - 1;
  }
  int lo = 0, hi = nsym;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (r * cum[mid] <= s.code)
      lo = mid;
    else
      hi = mid;
  }
  const uint32_t c0 = cum[lo], c1 = cum[lo + 1];
  s.code -= r * c0;
  s.range = r * (c1 - c0);
  while (s.range < kBot) {
    s.code = (s.code << 8) | rd.get(s, err);
    s.range <<= 8;
  }
  return lo;
}

// -log2(freq / 65536) of every (table, symbol), appended after the 64 CDF
// tables (see build_cdf_tables): one load per decoded symbol instead of an
// fp64 log2 on the lane's critical path.
__device__ __forceinline__ const double* bits_table(const uint32_t* cdf) {
  return reinterpret_cast<const double*>(cdf + kScales * (kSyms + 1));
}

// Decodes one value (escape + Exp-Golomb included); returns v, the table
// symbol k and the escape's extra bits (0 when k is not an escape). The
// lane's bit count is s.bits += bits_row[k] + then esc_bits, in symbol order.
template <class R>
__device__ int32_t dec_value_k(R& rd, LaneState& s, const uint32_t* cdf_row, int& k, int& esc_bits,
                               int& err) {
  k = dec_sym(rd, s, cdf_row, kSyms, err);
  esc_bits = 0;
  if (k < kEscLo) return k - 127;
  int nb = 0;
  while (dec_sym(rd, s, kBitCum, 2, err) == 0) {
    if (++nb > 31 || err) {
      err = 1;
      return 0;
    }
  }
  uint64_t x = 1;
  for (int i = 0; i < nb; ++i) x = (x << 1) | static_cast<uint64_t>(dec_sym(rd, s, kBitCum, 2, err));
  esc_bits = 2 * nb + 1;
  const long long m = static_cast<long long>(x) - 1 + 128;
  return static_cast<int32_t>(k == kEscLo ? -m : m);
}

template <class R>
__device__ int32_t dec_value(R& rd, LaneState& s, const uint32_t* cdf_row, const double* bits_row,
                             int& err) {
  int k, eb;
  const int32_t v = dec_value_k(rd, s, cdf_row, k, eb, err);
  s.bits += __ldg(bits_row + k);
  if (eb) s.bits += eb;
  return v;
}

// ------------------------------------------------------------ kernels -----
// Exclusive scan of one uint64 per thread over the block (warp shuffles, then
// the warp totals); ws is 33 shared words, ws[32] receives the block total.
// Integer sums, so the result does not depend on the order.
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t* ws) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t inc = v;
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t u = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    const uint64_t w = lane < nw ? ws[lane] : 0;
    uint64_t winc = w;
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t u = __shfl_up_sync(0xffffffffu, winc, d);
      if (lane >= d) winc += u;
    }
    if (lane < nw) ws[lane] = winc - w;
    if (lane == 31) ws[32] = winc;
  }
  __syncthreads();
  return ws[warp] + inc - v;
}

// One thread per lane, 128 lanes per block: each block first sums the
// lengths of all lanes before it (coalesced 2 / 4 B loads; the length table
// is L2-resident), then scans its own 128. Spreading the lanes over
// many SMs matters: the 6 scattered first-byte reads per lane are ~50k L2
// requests per frame, more than one SM's load path drains quickly.
__global__ void __launch_bounds__(128) lanes_init_kernel(const uint8_t* __restrict__ pl,
                                                         const uint32_t* __restrict__ len_p, int L,
                                                         uint32_t expect,
                                                         LaneState* __restrict__ lanes, int* status) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint64_t ws[33];
  const uint32_t len = *len_p;
  const int t = threadIdx.x;
  // header: L, symbol count, length-entry width w (2 or 4), then L lengths
  const uint32_t w = len >= 12 ? rd32(pl + 8) : 0u;
  const uint64_t hdr = 12u + static_cast<uint64_t>(w) * static_cast<uint32_t>(L);
  if (len < 12 || (w != 2 && w != 4) || len < hdr || rd32(pl) != static_cast<uint32_t>(L) ||
      rd32(pl + 4) != expect) {
    if (t == 0) atomicOr(status, 1);
    return;
  }
  const uint16_t* lens16 = reinterpret_cast<const uint16_t*>(pl + 12);  // 256 B-aligned payload
  const uint32_t* lens32 = reinterpret_cast<const uint32_t*>(pl + 12);
  auto lens = [&](int i) -> uint32_t { return w == 2 ? lens16[i] : lens32[i]; };
  const int l0 = blockIdx.x * blockDim.x;
  uint64_t before = 0;
  {
    int i = t;
    for (; i + 7 * 128 < l0; i += 8 * 128) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = lens(i + j * 128);
#pragma unroll
      for (int j = 0; j < 8; ++j) before += v[j];
    }
    for (; i < l0; i += 128) before += lens(i);
  }
  block_excl_scan(before, ws);
  before = ws[32];
  __syncthreads();  // ws is reused below
  const int l = l0 + t;
  const uint32_t ln = l < L ? lens(l) : 0u;
  const uint64_t off = hdr + before + block_excl_scan(ln, ws);
  if (l >= L) return;
  if (off + ln > len || ln < 4) {  // past the payload / shorter than the flush
    atomicOr(status, 1);
    // a dead lane the decoders can run over without leaving the payload
    LaneState s;
    s.pos = s.end = static_cast<uint32_t>(off < len ? off : len);
    s.range = kWin;
    s.code = 0;
    s.bits = 0.0;
    lanes[l] = s;
    return;
  }
  uint32_t byt[6];
#pragma unroll
  for (int b = 0; b < 6; ++b) byt[b] = static_cast<uint32_t>(b) < ln ? pl[off + b] : 0u;
  LaneState s;
  s.pos = static_cast<uint32_t>(off + 6);  // bytes past the lane's end are next_byte's implicit zeros
  s.end = static_cast<uint32_t>(off + ln);
  s.range = kWin;
  s.code = 0;
  s.bits = 0.0;
#pragma unroll
  for (int b = 0; b < 6; ++b) s.code = (s.code << 8) | byt[b];
  lanes[l] = s;
}

// Byte reservoir of one lane for the phase decoder: the lane's next bytes
// in a 64-bit register (cnt of them, the next one most significant), fed
// from 16 B-aligned windows; the following window is loaded as soon as the
// current one is entered, so its latency is hidden behind ~16 bytes of
// decoding. Reads may run up to 32 B past the lane's end (the payload
// buffer has that slack); bytes at or past `end` are masked to the implicit
// zeros of next_byte (two allowed, a third is an error).
struct Rsv {
  const uint8_t* pl;
  uint64_t bits;
  uint32_t cnt, wi, wb, pos, end;
  uint4 cur, nxt;
  __device__ __forceinline__ static uint32_t bswap(uint32_t w) { return __byte_perm(w, 0, 0x0123); }
  __device__ __forceinline__ uint32_t word(uint32_t i) const {
    return i < 2 ? (i == 0 ? cur.x : cur.y) : (i == 2 ? cur.z : cur.w);
  }
  __device__ __forceinline__ void advance() {
    const uint32_t enter = wi == 4;
    if (enter) {
      cur = nxt;
      wb += 16;
      wi = 0;
    }
    // the next window, loaded in place by an unconditional (predicated)
    // instruction with tied operands: as a plain conditional load the
    // compiler landed it in other registers and copied them at the loop back
    // edge, which turned every window prefetch into a full-latency stall of
    // the decode chain
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %5, 0;\n @p ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];\n}"
        : "+r"(nxt.x), "+r"(nxt.y), "+r"(nxt.z), "+r"(nxt.w)
        : "l"(pl + wb + 16), "r"(enter));
  }
  __device__ __forceinline__ void refill() {
    if (cnt < 2) {
      bits = (bits << 32) | bswap(word(wi));
      cnt += 4;
      ++wi;
      advance();
    }
  }
  __device__ __forceinline__ void init(const uint8_t* p, uint32_t pos0, uint32_t end0) {
    pl = p;
    pos = pos0;
    end = end0;
    wb = pos & ~15u;
    cur = __ldg(reinterpret_cast<const uint4*>(pl + wb));
    nxt = __ldg(reinterpret_cast<const uint4*>(pl + wb + 16));
    wi = (pos - wb) >> 2;
    const uint32_t skip = pos & 3u;
    bits = bswap(word(wi)) & (0xffffffffu >> (8 * skip));
    cnt = 4 - skip;
    ++wi;
    advance();
    refill();
  }
  // the next nb <= 2 bytes as one big-endian value
  __device__ __forceinline__ uint32_t take(uint32_t nb, int& err) {
    uint32_t v = static_cast<uint32_t>(bits >> (8 * (cnt - nb))) & ((1u << (8 * nb)) - 1u);
    if (pos + nb > end) {  // the lane's last bytes (rare)
      for (uint32_t i = 0; i < nb; ++i)
        if (pos + i >= end) {
          v &= ~(0xffu << (8 * (nb - 1 - i)));
          if (pos + i >= end + 2) err = 1;
        }
    }
    cnt -= nb;
    pos += nb;
    refill();
    return v;
  }
  __device__ __forceinline__ uint32_t get(LaneState&, int& err) { return take(1, err); }
};

// dec_sym over a 257-symbol table with its search index, same result: the
// target q = floor(code / r) (a float quotient, then one exact integer
// correction step each way: the float error is < 0.04 for q < 65536), a
// binary search only inside the symbols spanning q's 256-wide bucket
// (usually 1-2 candidates instead of 8 levels; closed form inside the
// tails' unit-frequency runs), and a branch-free
// renormalisation: the bytes dec_sym's `while (range < kBot)` loop reads,
// from the bit length of the new range (r >= 2^24, freq >= 1: at most 2).
__device__ __forceinline__ int dec_sym_rsv(Rsv& rs, LaneState& s, const uint32_t* cum,
                                           const uint16_t* lut, int& err) {
  const uint32_t r = static_cast<uint32_t>(s.range >> 16);
  const uint64_t lim = static_cast<uint64_t>(r) << 16;
  if (s.code >= lim) {
    err = 1;
    s.code = lim - 1;
  }
  uint32_t q = static_cast<uint32_t>(__fdividef(__ull2float_rz(s.code), __uint2float_rz(r)));
  q = min(q, 65535u);
  const uint64_t rq = static_cast<uint64_t>(r) * q;
  if (rq > s.code)
    --q;
  else if (rq + r <= s.code)
    ++q;
  const int b = static_cast<int>(q >> 8);
  const uint32_t e0 = lut[b], e1 = lut[b + 1];
  int lo = static_cast<int>(e0 & 0x7fffu);
  if (e0 & 0x8000u) {  // unit-frequency run: symbols past lo + 1 sit one per value
    const uint32_t c1 = cum[lo + 1];
    if (q >= c1) lo = min(lo + 1 + static_cast<int>(q - c1), static_cast<int>(e1 & 0x7fffu));
  } else {
    int hi = min(static_cast<int>(e1 & 0x7fffu) + 1, kSyms);
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (cum[mid] <= q)
        lo = mid;
      else
        hi = mid;
    }
  }
  const uint32_t c0 = cum[lo], c1 = cum[lo + 1];
  const uint64_t range = static_cast<uint64_t>(r) * (c1 - c0);
  const int bl = 64 - __clzll(static_cast<long long>(range));
  const uint32_t nb = bl > 40 ? 0u : static_cast<uint32_t>(48 - bl) >> 3;
  s.code = ((s.code - static_cast<uint64_t>(r) * c0) << (8 * nb)) | rs.take(nb, err);
  s.range = range << (8 * nb);
  return lo;
}

constexpr int kDecB = 16;  // symbols per lane gathered per batch (decode_phase)

__global__ void decode_phase_kernel(const uint8_t* __restrict__ pl, LaneState* __restrict__ lanes,
                                    int L, uint32_t o0_mod, int n, int per,
                                    const float* __restrict__ musig, int ldms, int sig_off,
                                    const float* __restrict__ scales, const uint32_t* __restrict__ cdf,
                                    const int* __restrict__ rows, int32_t* __restrict__ yhat, int C,
                                    int c0, __half* __restrict__ yhat16, int ld16, int* status,
                                    PhaseTaps taps) {
  // the 64 scale thresholds, the 64 cumulative tables (66 KB) and their
  // search indexes (33 KB) staged in shared memory: the sigma -> table and
  // symbol searches are dependent-load chains that otherwise run at L2
  // latency (one bulk async copy each: a per-thread copy loop serialises ~30
  // L2 round trips before the first symbol). The tables are built when the
  // handle is created, so they may be read before pdl_wait.
  extern __shared__ uint4 s_raw[];
  __shared__ uint64_t s_bar;
  uint32_t* s_cdf = reinterpret_cast<uint32_t*>(s_raw);
  uint16_t* s_lut = reinterpret_cast<uint16_t*>(s_cdf + kScales * (kSyms + 1));
  float* s_scales = reinterpret_cast<float*>(s_lut + kScales * kLutBuckets);
  constexpr uint32_t kCdfBytes = kScales * (kSyms + 1) * 4, kLutBytes = kScales * kLutBuckets * 2,
                     kScaleBytes = kScales * 4;
  static_assert(kCdfBytes % 16 == 0 && kLutBytes % 16 == 0 && kScaleBytes % 16 == 0,
                "bulk copies move 16 B multiples");
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    fence_mbar_init();
    fence_proxy_async_smem();
    mbar_expect_tx(&s_bar, kCdfBytes + kLutBytes + kScaleBytes);
    bulk_load(smem_u32(s_cdf), cdf, kCdfBytes, &s_bar);
    bulk_load(smem_u32(s_lut), sym_lut(cdf), kLutBytes, &s_bar);
    bulk_load(smem_u32(s_scales), scales, kScaleBytes, &s_bar);
  }
  __syncthreads();
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t total = static_cast<uint64_t>(n) * per;
  // first ordinal of lane l at or after o0, relative to o0 (o0_mod = o0 % L
  // from the host: no 64-bit division here)
  uint32_t i_first = static_cast<uint32_t>(l) + static_cast<uint32_t>(L) - o0_mod;
  if (i_first >= static_cast<uint32_t>(L)) i_first -= static_cast<uint32_t>(L);
  const bool active = l < L && i_first < total;
  // per-thread parameter slots in shared memory ([q][thread]: conflict-free):
  // the decode loop below is not unrolled, so its body exists once in the
  // binary (a 16x unrolled body overflowed the instruction cache)
  constexpr int kB = kDecB;
  const uint32_t ntot = static_cast<uint32_t>(total);
  const int Ldiv = L / per, Lmod = L - Ldiv * per;
  const double* bt = bits_table(cdf);
  int4* s_par = reinterpret_cast<int4*>(s_scales + kScales);  // {table | mu offset, mu, dst, dst16}
  int* s_out = reinterpret_cast<int*>(s_par + kB * blockDim.x);  // k | escape bits << 16
  double* s_cost = reinterpret_cast<double*>(s_out + kB * blockDim.x);  // [q][thread] symbol costs
  const int tid = threadIdx.x, nth = blockDim.x;
  auto batch_size = [&](uint32_t ib) {
    return min(kB, static_cast<int>((ntot - ib + L - 1) / static_cast<uint32_t>(L)));
  };
  // index part of a batch's parameters (symbol i -> (k, j) = divmod(i, per),
  // stepped by divmod(L, per): one division per batch): the mu/sigma offset
  // and the y_hat destinations, from the constant row table only
  auto batch_index = [&](uint32_t ib, int nq) {
    int k = static_cast<int>(ib) / per, j = static_cast<int>(ib) - k * per;
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      if (q > 0) {
        k += Ldiv;
        j += Lmod;
        if (j >= per) {
          j -= per;
          ++k;
        }
      }
      if (q < nq) s_par[q * nth + tid] = make_int4(k * ldms + j, 0, rows[k] * C + c0 + j, k * ld16 + c0 + j);
    }
  };
  // The lane state, payload bytes and the first batch's indexes are read
  // before the PDL wait: this grid starts once the head GEMM before it has
  // passed its own wait, so every earlier kernel (the previous phase, which
  // wrote the lane states, and the lane init) has completed. Only mu/sigma
  // come from the immediate predecessor.
  LaneState s;
  Rsv rs;
  if (active) {
    s = lanes[l];
    rs.init(pl, s.pos, s.end);
    batch_index(i_first, batch_size(i_first));
  }
  pdl_wait();
  pdl_trigger();
  mbar_wait(&s_bar, 0);
  // a malformed lane header (lanes_init) already failed the frame: decode nothing
  if (!active || (*reinterpret_cast<volatile int*>(status) & 1)) return;
  int err = 0;
  // the parameters (mu, table index) of a lane's next symbols do not depend
  // on the coder state: gather them in a batch (loads in flight together),
  // then run the sequential decode chain.
  // kB covers a lane's symbols of one full-frame phase (12 at 1080p with
  // 8192 lanes) in one batch. The bit-cost table loads are deferred to the
  // end of the batch (issued together, summed in symbol order) so their
  // latency is off the sequential decode chain.
  for (uint32_t ib = i_first; ib < ntot; ib += static_cast<uint32_t>(kB) * L) {
    const int nq = batch_size(ib);
    if (ib != i_first) batch_index(ib, nq);
    {
      float mu_f[kB], sg_f[kB];
      // all loads of the batch first (in flight together), then the table
      // searches: interleaving them exposes one load latency per symbol
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        if (q < nq) {
          const int off = s_par[q * nth + tid].x;
          mu_f[q] = musig[off];
          sg_f[q] = musig[off + sig_off];
        }
      }
      if (taps.mu) {  // the decoder's own entropy parameters (parity / BitStats taps)
#pragma unroll
        for (int q = 0; q < kB; ++q)
          if (q < nq) {
            const int dst = s_par[q * nth + tid].z;
            taps.mu[dst] = mu_f[q];
            taps.sigma[dst] = sg_f[q];
          }
      }
#pragma unroll
      for (int q = 0; q < kB; ++q)
        if (q < nq)
          *reinterpret_cast<int2*>(&s_par[q * nth + tid]) =
              make_int2(scale_index(s_scales, sg_f[q]), __float2int_rn(mu_f[q]));
    }
#pragma unroll 1
    for (int q = 0; q < nq; ++q) {
      const int4 pr = s_par[q * nth + tid];
      const int k = dec_sym_rsv(rs, s, s_cdf + pr.x * (kSyms + 1), s_lut + pr.x * kLutBuckets, err);
      int eb = 0;
      int32_t v = k - 127;
      if (k >= kEscLo) {  // escape: Exp-Golomb magnitude (rare)
        int nb = 0;
        bool bad = false;
        while (dec_sym(rs, s, kBitCum, 2, err) == 0) {
          if (++nb > 31 || err) {
            bad = true;
            break;
          }
        }
        if (bad) {
          err = 1;
          v = 0;
        } else {
          uint64_t x = 1;
          for (int i = 0; i < nb; ++i) x = (x << 1) | static_cast<uint64_t>(dec_sym(rs, s, kBitCum, 2, err));
          eb = 2 * nb + 1;
          const long long m = static_cast<long long>(x) - 1 + 128;
          v = static_cast<int32_t>(k == kEscLo ? -m : m);
        }
      }
      s_out[q * nth + tid] = k | (eb << 16);
      // this symbol's cost (fp64, global) fetched into smem while the chain
      // continues; summed after the chain in symbol order
      cp_async_8(smem_u32(s_cost + q * nth + tid), bt + pr.x * kSyms + k);
      const int32_t y = v + pr.y;
      // a y_hat the encoder cannot have produced (|y_hat| > kYhatMax) marks
      // the stream corrupt
      if (y > taps.ymax || y < -taps.ymax) err = 1;
      yhat[pr.z] = y;
      if (yhat16) yhat16[pr.w] = __int2half_rn(y);
      // a lane that ran past its end stops here: no further reads past the
      // payload (the frame fails with status 2)
      if (err) break;
    }
    if (err) break;
    // bit costs: copied during the chain, summed in symbol order
    cp_async_wait_all();
    double cost[kB];
    int ebs[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      cost[q] = 0.0;
      ebs[q] = 0;
      if (q < nq) {
        ebs[q] = s_out[q * nth + tid] >> 16;
        cost[q] = s_cost[q * nth + tid];
      }
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      if (q >= nq) break;
      s.bits += cost[q];
      if (ebs[q]) s.bits += ebs[q];
    }
    if (taps.bits) {
#pragma unroll
      for (int q = 0; q < kB; ++q)
        if (q < nq) taps.bits[s_par[q * nth + tid].z] = cost[q] + static_cast<double>(ebs[q]);
    }
  }
  cp_async_wait_all();  // (an erroring lane left the batch with copies in flight)
  s.pos = rs.pos;
  lanes[l] = s;
  if (err) atomicOr(status, 2);
}

__global__ void decode_hyper_kernel(const uint8_t* __restrict__ pl, LaneState* __restrict__ lanes,
                                    int L, int n, int per_ch, const float* __restrict__ loc,
                                    const float* __restrict__ scale, const float* __restrict__ scales,
                                    const uint32_t* __restrict__ cdf, int32_t* __restrict__ zhat,
                                    int* status) {
  pdl_wait();
  pdl_trigger();
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L || (*status & 1)) return;
  LaneState s = lanes[l];
  int err = 0;
  for (int i = l; i < n && !err; i += L) {
    const int ch = i / per_ch;
    const int idx = scale_index(scales, scale[ch]);
    ByteDirect rd{pl};
    const int32_t v = dec_value(rd, s, cdf + idx * (kSyms + 1), bits_table(cdf) + idx * kSyms, err);
    zhat[i] = v + __float2int_rn(loc[ch]);
  }
  lanes[l] = s;
  if (err) atomicOr(status, 2);
}

// Escape bits of a coded value (Exp-Golomb(0) of |v| - 128, 0 in range).
__device__ __forceinline__ int escape_bits(int64_t v) {
  if (v >= -127 && v <= 127) return 0;
  const uint64_t x = static_cast<uint64_t>(v < 0 ? -v : v) - 128 + 1;
  return 2 * (63 - __clzll(static_cast<long long>(x))) + 1;
}

__global__ void quantize_phase_kernel(const float* __restrict__ musig, int ldms, int sig_off, int n,
                                      int per, uint64_t o0, const int* __restrict__ rows,
                                      const int32_t* __restrict__ yhat, int C, int c0,
                                      const float* __restrict__ scales, const uint32_t* __restrict__ cdf,
                                      int32_t* __restrict__ sym_v, uint8_t* __restrict__ sym_idx,
                                      __half* __restrict__ yhat16, int ld16, PhaseTaps taps,
                                      int* status) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * per) return;
  const int k = i / per, j = i - k * per;
  const float mu = musig[static_cast<size_t>(k) * ldms + j];
  const float sg = musig[static_cast<size_t>(k) * ldms + sig_off + j];
  const size_t e = static_cast<size_t>(rows[k]) * C + c0 + j;
  const int32_t y = yhat[e];
  // the coded value must stay in the escape code's 32-bit range (a mean
  // that is not finite, from a y_hat outside the supported range, lands here)
  const int64_t v = static_cast<int64_t>(y) - static_cast<int64_t>(__float2ll_rn(mu));
  if (y > kYhatMax || y < -kYhatMax || !(fabsf(mu) < 1.0e9f) || v > INT32_MAX - 128 ||
      v < -(INT32_MAX - 128))
    atomicOr(status, 16);
  const int idx = scale_index(scales, sg);
  sym_v[o0 + i] = static_cast<int32_t>(v);
  sym_idx[o0 + i] = static_cast<uint8_t>(idx);
  if (yhat16) yhat16[static_cast<size_t>(k) * ld16 + c0 + j] = __int2half_rn(y);
  if (taps.mu) {
    taps.mu[e] = mu;
    taps.sigma[e] = sg;
  }
  if (taps.bits) {
    const int ks = v < -127 ? kEscLo : (v > 127 ? kEscHi : static_cast<int>(v) + 127);
    taps.bits[e] = bits_table(cdf)[idx * kSyms + ks] + static_cast<double>(escape_bits(v));
  }
}

// One thread per (group, position): the group's Cg symbol costs in channel
// order (a fixed order: BitStats are bitwise identical on both sides).
__global__ void bitstats_kernel(const double* __restrict__ sym_bits, int C, int row0, int npos,
                                int N, int Cg, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N * npos) return;
  const int g = i / npos, p = i - g * npos;
  const double* b = sym_bits + static_cast<size_t>(row0 + p) * C + g * Cg;
  double acc = 0.0;
  for (int c = 0; c < Cg; ++c) acc += b[c];
  out[i] = acc;
}

__global__ void quantize_hyper_kernel(const int32_t* __restrict__ zhat, int n, int per_ch,
                                      const float* __restrict__ loc, const float* __restrict__ scale,
                                      const float* __restrict__ scales, int32_t* __restrict__ sym_v,
                                      uint8_t* __restrict__ sym_idx) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ch = i / per_ch;
  sym_v[i] = zhat[i] - __float2int_rn(loc[ch]);
  sym_idx[i] = static_cast<uint8_t>(scale_index(scales, scale[ch]));
}

struct Enc {
  uint64_t low, range;
  uint32_t n;
  bool overflow;
  uint8_t* out;
  uint32_t cap;
  __device__ void carry() {
    for (uint32_t i = n; i-- > 0;)
      if (++out[i] != 0) break;
  }
  __device__ void emit(uint8_t b) {
    if (n < cap)
      out[n++] = b;
    else
      overflow = true;
  }
  __device__ void put(uint32_t cum, uint32_t freq) {
    const uint64_t r = range >> 16;
    low += r * cum;
    range = r * freq;
    if (low > kWin) {
      low &= kWin;
      carry();
    }
    while (range < kBot) {
      emit(static_cast<uint8_t>(low >> 40));
      low = (low << 8) & kWin;
      range <<= 8;
    }
  }
};

__global__ void encode_lanes_kernel(const int32_t* __restrict__ sym_v, const uint8_t* __restrict__ sym_idx,
                                    uint64_t n, int L, const uint32_t* __restrict__ cdf,
                                    uint8_t* __restrict__ out, uint32_t cap, uint32_t* __restrict__ lens,
                                    double* __restrict__ bits, int* status) {
  pdl_wait();
  pdl_trigger();
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  Enc e{0, kWin, 0, false, out + static_cast<size_t>(l) * cap, cap};
  double b = 0.0;
  for (uint64_t o = l; o < n; o += L) {
    const int32_t v = sym_v[o];
    const uint32_t* c = cdf + sym_idx[o] * (kSyms + 1);
    const int k = v < -127 ? kEscLo : (v > 127 ? kEscHi : v + 127);
    const uint32_t c0 = __ldg(c + k), c1 = __ldg(c + k + 1);
    e.put(c0, c1 - c0);
    b += __ldg(bits_table(cdf) + sym_idx[o] * kSyms + k);
    if (k >= kEscLo) {
      const uint64_t x = static_cast<uint64_t>(v < 0 ? -static_cast<int64_t>(v) : v) - 128 + 1;
      int nb = 0;
      while ((x >> (nb + 1)) != 0) ++nb;
      for (int i = 0; i < nb; ++i) e.put(0u, 32768u);
      for (int i = nb; i >= 0; --i) e.put(((x >> i) & 1) ? 32768u : 0u, 32768u);
      b += 2 * nb + 1;
    }
  }
  uint64_t v = (e.low + 0xFFFF) & ~uint64_t{0xFFFF};
  if (v > kWin) {
    v &= kWin;
    e.carry();
  }
  for (int sh = 40; sh >= 16; sh -= 8) e.emit(static_cast<uint8_t>(v >> sh));
  lens[l] = e.n;
  bits[l] = b;
  if (e.overflow) atomicOr(status, 4);
}

__global__ void sum_bits_kernel(const double* __restrict__ v, int stride, int L, double* out) {
  pdl_wait();
  pdl_trigger();
  __shared__ double part[256];
  const int t = threadIdx.x;
  const int per = (L + 255) / 256;
  double acc = 0.0;
  for (int l = t * per; l < min(L, (t + 1) * per); ++l) acc += v[static_cast<size_t>(l) * stride];
  part[t] = acc;
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
    for (int i = 0; i < 256; ++i) s += part[i];
    *out = s;
  }
}

inline int blocks(long n, int t = 128) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

void build_cdf_tables(float* scales, uint32_t* cdf, cudaStream_t st, int laplace) {
  launch_k(build_cdf_kernel, dim3(1), dim3(kScales), 0, st, scales, cdf, laplace);
  PSWA_LAUNCH_CHECK();
}

void lanes_init(const uint8_t* payload, const uint32_t* len, int lanes, uint32_t expect_count,
                LaneState* st_lanes, int* status, cudaStream_t st) {
  launch_k(lanes_init_kernel, dim3((lanes + 127) / 128), dim3(128), 0, st, payload, len, lanes, expect_count,
           st_lanes, status);
  PSWA_LAUNCH_CHECK();
}

void lanes_decode_phase(const uint8_t* payload, LaneState* lanes, int L, uint64_t o0, int n,
                        int per, const float* musig, int ldms, int sig_off, const float* scales,
                        const uint32_t* cdf, const int* rows, int32_t* yhat, int C, int c0,
                        __half* yhat16, int ld16, int* status, cudaStream_t st, PhaseTaps taps) {
  if (n <= 0) return;
  constexpr int smem = kScales * (kSyms + 1) * 4 + kScales * kLutBuckets * 2 + kScales * 4 +
                       kDecB * 128 * (16 + 4 + 8);
  static const bool attr = [] {
    PSWA_CUDA(cudaFuncSetAttribute(decode_phase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return true;
  }();
  (void)attr;
  launch_k(decode_phase_kernel, dim3(blocks(L)), dim3(128), smem, st, payload, lanes, L,
           static_cast<uint32_t>(o0 % static_cast<uint64_t>(L)), n, per, musig, ldms,
                                                  sig_off, scales, cdf, rows, yhat, C, c0, yhat16,
                                                  ld16, status, taps);
  PSWA_LAUNCH_CHECK();
}

void lanes_decode_hyper(const uint8_t* payload, LaneState* lanes, int L, int n, int per_ch,
                        const float* loc, const float* scale, const float* scales,
                        const uint32_t* cdf, int32_t* zhat, int* status, cudaStream_t st) {
  launch_k(decode_hyper_kernel, dim3(blocks(L)), dim3(128), 0, st, payload, lanes, L, n, per_ch, loc, scale, scales,
                                                  cdf, zhat, status);
  PSWA_LAUNCH_CHECK();
}

void quantize_phase(const float* musig, int ldms, int sig_off, int n, int per, uint64_t o0,
                    const int* rows, const int32_t* yhat, int C, int c0, const float* scales,
                    const uint32_t* cdf, int32_t* sym_v, uint8_t* sym_idx, __half* yhat16, int ld16,
                    PhaseTaps taps, int* status, cudaStream_t st) {
  if (n <= 0) return;
  launch_k(quantize_phase_kernel, dim3(blocks(static_cast<long>(n) * per, 256)), dim3(256), 0, st,
           musig, ldms, sig_off, n, per, o0, rows, yhat, C, c0, scales, cdf, sym_v, sym_idx, yhat16,
           ld16, taps, status);
  PSWA_LAUNCH_CHECK();
}

void bitstats_reduce(const double* sym_bits, int C, int row0, int npos, int N, int Cg, double* out,
                     cudaStream_t st) {
  if (npos <= 0) return;
  launch_k(bitstats_kernel, dim3(blocks(static_cast<long>(N) * npos, 256)), dim3(256), 0, st,
           sym_bits, C, row0, npos, N, Cg, out);
  PSWA_LAUNCH_CHECK();
}

void quantize_hyper(const int32_t* zhat, int n, int per_ch, const float* loc, const float* scale,
                    const float* scales, int32_t* sym_v, uint8_t* sym_idx, cudaStream_t st) {
  launch_k(quantize_hyper_kernel, dim3(blocks(n, 256)), dim3(256), 0, st, zhat, n, per_ch, loc, scale, scales, sym_v,
                                                        sym_idx);
  PSWA_LAUNCH_CHECK();
}

void lanes_encode(const int32_t* sym_v, const uint8_t* sym_idx, uint64_t n, int L,
                  const uint32_t* cdf, uint8_t* out, uint32_t cap, uint32_t* lens, double* bits,
                  int* status, cudaStream_t st) {
  launch_k(encode_lanes_kernel, dim3(blocks(L)), dim3(128), 0, st, sym_v, sym_idx, n, L, cdf, out, cap, lens, bits,
                                                  status);
  PSWA_LAUNCH_CHECK();
}

namespace {
__global__ void accumulate_status_kernel(const int* status, int* sticky) {
  pdl_wait();
  pdl_trigger();
  if (*status) atomicOr(sticky, *status);
}
}  // namespace

void accumulate_status(const int* status, int* sticky, cudaStream_t st) {
  launch_k(accumulate_status_kernel, dim3(1), dim3(1), 0, st, status, sticky);
  PSWA_LAUNCH_CHECK();
}

void sum_lane_bits(const LaneState* lanes, int L, double* out, cudaStream_t st) {
  launch_k(sum_bits_kernel, dim3(1), dim3(256), 0, st, &lanes[0].bits, static_cast<int>(sizeof(LaneState) / 8), L,
                                     out);
  PSWA_LAUNCH_CHECK();
}

void sum_doubles(const double* v, int L, double* out, cudaStream_t st) {
  launch_k(sum_bits_kernel, dim3(1), dim3(256), 0, st, v, 1, L, out);
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev

namespace pswa_dev {
namespace {
__global__ void pack_offsets_kernel(const uint32_t* __restrict__ lens, int L, uint32_t count,
                                    uint8_t* __restrict__ payload, uint64_t cap,
                                    unsigned long long* total, uint64_t* __restrict__ offs, int* status) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint64_t ws[33];
  __shared__ uint32_t longest;
  const int t = threadIdx.x;
  const int per = (L + blockDim.x - 1) / blockDim.x;
  const int l0 = t * per, l1 = min(L, l0 + per);
  if (t == 0) longest = 0;
  __syncthreads();
  uint64_t acc = 0;
  uint32_t mx = 0;
  for (int l = l0; l < l1; ++l) {
    acc += lens[l];
    mx = max(mx, lens[l]);
  }
  if (mx) atomicMax(&longest, mx);
  const uint64_t excl = block_excl_scan(acc, ws);  // (its barriers publish `longest`)
  // length entries of 2 bytes when every lane is shorter than 64 KiB
  const uint32_t w = longest < 65536u ? 2u : 4u;
  const uint64_t hdr = 12 + static_cast<uint64_t>(w) * L;
  if (t == 0) {
    *total = hdr + ws[32];
    if (hdr + ws[32] > cap) atomicOr(status, 8);
  }
  uint64_t off = hdr + excl;
  for (int l = l0; l < l1; ++l) {
    offs[l] = off;
    off += lens[l];
  }
  auto wr = [&](uint64_t at, uint32_t v, uint32_t nb) {
    if (at + nb <= cap)
      for (uint32_t b = 0; b < nb; ++b) payload[at + b] = static_cast<uint8_t>(v >> (8 * b));
  };
  if (t == 0) {
    wr(0, static_cast<uint32_t>(L), 4);
    wr(4, count, 4);
    wr(8, w, 4);
  }
  for (int l = l0; l < l1; ++l) wr(12 + static_cast<uint64_t>(w) * l, lens[l], w);
}

__global__ void pack_copy_kernel(const uint8_t* __restrict__ enc, uint32_t cap_lane,
                                 const uint32_t* __restrict__ lens, const uint64_t* __restrict__ offs,
                                 int L, uint8_t* __restrict__ payload, uint64_t cap) {
  pdl_wait();
  pdl_trigger();
  const int l = blockIdx.x;
  if (l >= L) return;
  const uint64_t off = offs[l];
  const uint32_t n = lens[l];
  if (off + n > cap) return;
  const uint8_t* src = enc + static_cast<size_t>(l) * cap_lane;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) payload[off + i] = src[i];
}
}  // namespace

void lanes_pack(const uint8_t* enc, uint32_t cap, const uint32_t* lens, int L, uint32_t count,
                uint8_t* payload, uint64_t payload_cap, unsigned long long* total, uint64_t* offs,
                int* status, cudaStream_t st) {
  launch_k(pack_offsets_kernel, dim3(1), dim3(1024), 0, st, lens, L, count, payload, payload_cap, total, offs, status);
  PSWA_LAUNCH_CHECK();
  launch_k(pack_copy_kernel, dim3(L), dim3(64), 0, st, enc, cap, lens, offs, L, payload, payload_cap);
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
