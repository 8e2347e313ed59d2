// Tensor-core windowed attention (head_dim 32, 7x7 window), transposed
// FlashAttention-2 formulation: per warp 8 queries, scores computed as
// S^T = K . Q^T (keys on the MMA's M side, queries on N), probabilities moved
// into the PV operand with movmatrix, O^T = V^T . P^T; mma.sync m16n8k16, fp16
// operands, fp32 accumulation, masks and bias from a per-shape table.
//
// Why transposed. m16n8k16 needs 16 rows on M but only 8 columns on N. With
// the keys on M, a warp owns 8 queries, which fit in a compact 2x4 block
// (context) or the 8 step-t positions of a 4x8 block (step batches). The key
// union a warp scans shrinks accordingly:
//   * context, 2x4 queries: an 8x10 band, 80 keys per slot for 49 in-window
//     (61%; the previous 1x16-strip, 16-query layout scanned 160);
//   * step batches: a 10x14 band, keys sorted by wavefront step class so the
//     masked classes (<= t for S1/S2 self, < t for the
//     accumulator) are never scanned: step 0 scans 48 keys, not 140.
// Work is a list of CTA tiles x head groups: the CTA walks (head, slot)
// stages; each stage's K/V halo of its query rectangle is one pair of 4D TMA
// boxes (zero-filled outside the grid, SWIZZLE_128B) issued by one thread
// and double-buffered so the next halo loads while this one is consumed.
// Each warp walks only its band, in 16-key chunks, two passes per slot
// (scores + max, then exp + PV) so the softmax reductions happen once per
// slot rather than once per chunk.
//
// Semantics match SPEC.md:221-256 and the oracle: out-of-grid keys are
// masked (not padded), the learned per-offset bias is added to the scaled
// score, softmax in fp32, a query with no allowed key outputs zeros.
#include <cfloat>
#include <cstdlib>

#include "check.h"
#include "kernels.h"
#include "launch.cuh"
#include "ptx.cuh"

namespace pswa_dev {

namespace {

constexpr int kHD = 32;  // head dim handled by this kernel
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
// 8x8 b16 transpose across the warp (C-fragment layout in, transposed out)
__device__ __forceinline__ uint32_t movtrans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
// Byte offset of (halo key, 16 B chunk) in a [key][32 halves] halo buffer
// written by TMA with SWIZZLE_64B (64 B rows): address bits [4:5] ^= bits
// [7:8]. With the band orders used (column-major context bands over a
// 23-wide halo, step-class-sorted bands over a 24-wide halo) the 8 rows of an
// ldmatrix phase land on distinct 16 B bank groups (context) or at most
// 2-way (steps).
__device__ __forceinline__ uint32_t swz(int key, int chunk) {
  const uint32_t off = static_cast<uint32_t>(key * 64 + chunk * 16);
  return off ^ (((off >> 7) & 3u) << 4);
}

struct AttnArgs {
  const __half* q;
  int ldq;
  const int32_t* tiles;
  int d;
  int wt;  // > 0: 3D context window over wt slots
  const __half* tables;  // [heads][nsl][nbk][8] score offsets (build_score_tables)
  int nsl;              // slot offsets per head in `tables` (wt for 3D, 1 for 2D)
  __half* out;
  int ldo;
  AttnShape shape;
  int hw;      // halo width (keys per halo row)
  int kbuf;    // bytes of one K (or V) halo buffer (1024-aligned)
  int dbuf;    // double-buffer the (head, slot) halos
  int hpc;     // heads per CTA (pipelined)
};

// NP passes of up to PC 16-key chunks per (head, slot) stage; the online
// softmax carries across passes like across slots, so the register
// footprint is that of one pass. NP = 2 keeps 2 CTAs per SM: forcing 3
// (80 registers, 68 B of spills) measured slower (15.7 -> 18.5 us).
// QW = queries per warp: 8 (one MMA N tile) or 16 (two N tiles sharing every
// K / V fragment: a 4x4 query block scans a 10x10 key band, 6.25 keys per
// query against 10 for the 2x4 block of QW = 8).
template <int QW>
constexpr int pass_chunks() { return QW == 16 ? 4 : 5; }
// (Step tiles recomputing their ldmatrix row keys per chunk to fit 3 CTAs
// per SM at 76 registers measured 15.9 vs 15.6 us per launch: reverted.)
template <int NP, int QW>
__global__ void __launch_bounds__(256, (NP == 1 && QW == 8) ? 3 : 2)
    window_attn_t8_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap kvmap) {
  constexpr int PC = pass_chunks<QW>();
  constexpr int NT = QW / 8;       // MMA N tiles (8 queries each)
  constexpr int WI = 2 + QW;       // tile ints per warp
  constexpr int NCH = NP * PC;     // chunk slots held in registers (row keys)
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid x = head group (fastest in dispatch order), y = tile: a tile's head
  // groups launch together, so tile order (heaviest first) is dispatch order
  const int h0 = blockIdx.x * a.hpc;  // this CTA's heads: [h0, h0 + hpc)
  const int32_t* T = a.tiles + blockIdx.y * kAttnTileInts;
  const int hy0 = T[0], hx0 = T[1], HR = T[2], sl = T[3], nw = T[4];
  const int nslots = a.wt > 0 ? min(sl + 1, a.wt) : 1;
  const int j0 = sl - nslots + 1;
  const int nstages = a.hpc * nslots;  // pipeline over (head, slot)
  const int nbuf = a.dbuf ? 2 : 1;
  const uint32_t sraw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t sbase = (sraw + 1023u) & ~1023u;  // swizzled TMA boxes: 1024 B aligned
  uint8_t* smem = smem_raw + (sbase - sraw);
  // [2][kAttnMaxBandKeys][QW] fp16 score offsets (128 B aligned), then barriers, band keys
  __half* stbl0 = reinterpret_cast<__half*>(smem + nbuf * 2 * a.kbuf);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stbl0 + 2 * kAttnMaxBandKeys * QW);  // [2] stage-full
  int16_t* sbk = reinterpret_cast<int16_t*>(bars + 2);  // band key: row<<8 | col
  const int nbk = a.shape.nbk;
  const uint32_t box_bytes = static_cast<uint32_t>(HR * a.hw * 64);
  const uint32_t tbl_bytes = static_cast<uint32_t>(nbk * QW * 2);
  const CUtensorMap* kvm = &kvmap;  // param-space address (never copied to local memory)

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    tma_prefetch(kvm);
  }
  // the band keys are constants: safe to read before the PDL wait
  for (int i = threadIdx.x; i < nbk; i += blockDim.x) sbk[i] = a.shape.bkey[i];
  pdl_wait();  // K/V and Q come from the previous kernels
  pdl_trigger();
  __syncthreads();

  // one elected thread stages (head h, slot j): two 4D TMA boxes (K, V) and
  // the (head, slot offset) score-offset table, on one mbarrier
  auto stage = [&](int h, int j, int buf) {
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();  // prior ldmatrix reads of this buffer before the overwrite
      const uint32_t kb = sbase + buf * 2 * a.kbuf;
      mbar_expect_tx(&bars[buf], 2 * box_bytes + tbl_bytes);
      tma_load_4d(kb, kvm, &bars[buf], h * kHD, hx0, hy0, j);
      tma_load_4d(kb + a.kbuf, kvm, &bars[buf], a.d + h * kHD, hx0, hy0, j);
      const int so = a.wt > 0 ? j - sl + a.wt - 1 : 0;
      if (tbl_bytes)
        bulk_load(static_cast<uint32_t>(__cvta_generic_to_shared(stbl0 + buf * kAttnMaxBandKeys * QW)),
                  a.tables + (static_cast<size_t>(h) * a.nsl + so) * nbk * QW, tbl_bytes, &bars[buf]);
    }
  };
  uint32_t phase = 0;  // bit b: parity of the next completion of bars[b]
  auto wait_buf = [&](int buf) {
    mbar_wait(&bars[buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;
  };
  stage(h0, j0, 0);

  const int32_t* Wd = T + 8 + warp * WI;
  const int br = warp < nw ? Wd[0] : 0, bc = warp < nw ? Wd[1] : 0;  // band origin in the halo
  int qrow[NT];  // query 8n + lane/4 of N tile n (B-operand column)
#pragma unroll
  for (int n = 0; n < NT; ++n) qrow[n] = warp < nw ? Wd[2 + 8 * n + (lane >> 2)] : -1;
  bool any_q = false;
#pragma unroll
  for (int n = 0; n < NT; ++n) any_q = any_q || qrow[n] >= 0;
  const bool live = __any_sync(0xffffffffu, any_q);

  // per-lane ldmatrix row keys (K: non-transposed A operand; V: transposed,
  // read per chunk) and the in-grid bits of the two score rows per chunk
  const int nch = nbk / 16;
  auto halo_key = [&](int bk) {
    const int v = sbk[bk];
    return (br + (v >> 8)) * a.hw + bc + (v & 255);
  };
  int hk[NCH], hv[NCH];
  uint32_t inb = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    hk[c] = hv[c] = 0;
    if (c < nch) {
      hk[c] = halo_key(c * 16 + (lane & 7) + ((lane >> 3) & 1) * 8);
      hv[c] = halo_key(c * 16 + (lane & 7) + ((lane >> 4) & 1) * 8);
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int v = sbk[c * 16 + (lane >> 2) + 8 * rr];
        const int ky = hy0 + br + (v >> 8), kx = hx0 + bc + (v & 255);
        if (ky >= 0 && ky < a.shape.H && kx >= 0 && kx < a.shape.W) inb |= 1u << (2 * c + rr);
      }
    }
  }
  const int qc = (lane & 3) * 2;                         // my two query columns in C fragments
  const float qscale = 0.17677669529663687f * kLog2e;    // log2(e) / sqrt(32)
  uint32_t qb[NT][2][2];
  float o[NT][2][4];
  float m0[NT], m1[NT], l0[NT], l1[NT];

  int hi = 0, js = 0;  // stage st = (head h0 + hi, slot j0 + js)
  for (int st = 0; st < nstages; ++st) {
    const int h = h0 + hi, j = j0 + js;
    const int buf = nbuf == 2 ? (st & 1) : 0;
    if (nbuf == 1 && st > 0) stage(h, j, 0);  // previous stage fully consumed (barrier below)
    if (nbuf == 2 && st + 1 < nstages) {
      const bool wrap = js + 1 == nslots;  // prefetch the next (head, slot) halo
      stage(wrap ? h + 1 : h, wrap ? j0 : j + 1, buf ^ 1);
    }
    if (js == 0) {  // new head: my queries' fragments, fresh softmax state
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const __half* qp = a.q + static_cast<size_t>(qrow[n] < 0 ? 0 : qrow[n]) * a.ldq + h * kHD + qc;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          qb[n][ks][0] = qrow[n] >= 0 ? *reinterpret_cast<const uint32_t*>(qp + ks * 16) : 0u;
          qb[n][ks][1] = qrow[n] >= 0 ? *reinterpret_cast<const uint32_t*>(qp + ks * 16 + 8) : 0u;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) o[n][i][e] = 0.0f;
        m0[n] = m1[n] = -INFINITY;
        l0[n] = l1[n] = 0.0f;
      }
    }
    wait_buf(buf);  // halo and score-offset table of this stage landed
    const uint32_t sK = sbase + buf * 2 * a.kbuf, sV = sK + a.kbuf;
    const __half* stbl = stbl0 + buf * kAttnMaxBandKeys * QW;
    if (live) {
#pragma unroll
      for (int ps = 0; ps < NP; ++ps) {
        if (ps * PC >= nch) break;
        // pass 1: scores and their per-query max over these chunks; each K
        // fragment feeds the NT query tiles
        float s[PC][NT][4];
        float mx0[NT], mx1[NT];
#pragma unroll
        for (int n = 0; n < NT; ++n) mx0[n] = mx1[n] = -INFINITY;
#pragma unroll
        for (int ci = 0; ci < PC; ++ci) {
          const int c = ps * PC + ci;
          if (c < nch) {
            float acc[NT][4];
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
              for (int e = 0; e < 4; ++e) acc[n][e] = 0.0f;
            uint32_t fa[4];
            ldsm_x4(sK + swz(hk[c], lane >> 4), fa);
#pragma unroll
            for (int n = 0; n < NT; ++n) mma16816(acc[n], fa, qb[n][0][0], qb[n][0][1]);
            ldsm_x4(sK + swz(hk[c], (lane >> 4) + 2), fa);
#pragma unroll
            for (int n = 0; n < NT; ++n) mma16816(acc[n], fa, qb[n][1][0], qb[n][1][1]);
            const int r0 = c * 16 + (lane >> 2);
            const bool k0 = (inb >> (2 * c)) & 1u, k1 = (inb >> (2 * c + 1)) & 1u;
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              const float2 t0 = __half22float2(*reinterpret_cast<const __half2*>(stbl + r0 * QW + 8 * n + qc));
              const float2 t1 =
                  __half22float2(*reinterpret_cast<const __half2*>(stbl + (r0 + 8) * QW + 8 * n + qc));
              s[ci][n][0] = k0 ? fmaf(acc[n][0], qscale, t0.x) : -INFINITY;
              s[ci][n][1] = k0 ? fmaf(acc[n][1], qscale, t0.y) : -INFINITY;
              s[ci][n][2] = k1 ? fmaf(acc[n][2], qscale, t1.x) : -INFINITY;
              s[ci][n][3] = k1 ? fmaf(acc[n][3], qscale, t1.y) : -INFINITY;
              mx0[n] = fmaxf(mx0[n], fmaxf(s[ci][n][0], s[ci][n][2]));
              mx1[n] = fmaxf(mx1[n], fmaxf(s[ci][n][1], s[ci][n][3]));
            }
          }
        }
        float ms0[NT], ms1[NT];
#pragma unroll
        for (int n = 0; n < NT; ++n) {
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) {
            mx0[n] = fmaxf(mx0[n], __shfl_xor_sync(0xffffffffu, mx0[n], off));
            mx1[n] = fmaxf(mx1[n], __shfl_xor_sync(0xffffffffu, mx1[n], off));
          }
          const float mn0 = fmaxf(m0[n], mx0[n]), mn1 = fmaxf(m1[n], mx1[n]);
          const float al0 = mn0 == -INFINITY ? 1.0f : ex2(m0[n] - mn0);  // ex2(-inf) = 0
          const float al1 = mn1 == -INFINITY ? 1.0f : ex2(m1[n] - mn1);
          m0[n] = mn0;
          m1[n] = mn1;
          // exp offsets: a query with no allowed key yet keeps m = -inf; use
          // 0 so that ex2(-inf - 0) = 0 instead of NaN
          ms0[n] = mn0 == -INFINITY ? 0.0f : mn0;
          ms1[n] = mn1 == -INFINITY ? 0.0f : mn1;
          l0[n] *= al0;
          l1[n] *= al1;
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            o[n][mt][0] *= al0;
            o[n][mt][1] *= al1;
            o[n][mt][2] *= al0;
            o[n][mt][3] *= al1;
          }
        }
        // pass 2: probabilities (fp16) and O^T += V^T P^T; each V fragment
        // feeds the NT query tiles
#pragma unroll
        for (int ci = 0; ci < PC; ++ci) {
          const int c = ps * PC + ci;
          if (c < nch) {
            uint32_t b0[NT], b1[NT];
#pragma unroll
            for (int n = 0; n < NT; ++n) {
              const float p0 = ex2(s[ci][n][0] - ms0[n]), p1 = ex2(s[ci][n][1] - ms1[n]);
              const float p2 = ex2(s[ci][n][2] - ms0[n]), p3 = ex2(s[ci][n][3] - ms1[n]);
              l0[n] += p0 + p2;
              l1[n] += p1 + p3;
              b0[n] = movtrans(pack_h2(p0, p1));
              b1[n] = movtrans(pack_h2(p2, p3));
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              uint32_t fv[4];
              ldsm_x4_t(sV + swz(hv[c], ((lane >> 3) & 1) + 2 * mt), fv);
#pragma unroll
              for (int n = 0; n < NT; ++n) mma16816(o[n][mt], fv, b0[n], b1[n]);
            }
          }
        }
      }
      if (js == nslots - 1) {  // head done: normalise and store
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          float t0 = l0[n], t1 = l1[n];
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) {
            t0 += __shfl_xor_sync(0xffffffffu, t0, off);
            t1 += __shfl_xor_sync(0xffffffffu, t1, off);
          }
          const float inv0 = t0 > 0.0f ? 1.0f / t0 : 0.0f;
          const float inv1 = t1 > 0.0f ? 1.0f / t1 : 0.0f;
          // O^T blocks (8 dims x 8 queries) -> row-major O rows via movmatrix
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {
              const uint32_t v = movtrans(pack_h2(o[n][mt][2 * hb] * inv0, o[n][mt][2 * hb + 1] * inv1));
              if (qrow[n] >= 0)
                *reinterpret_cast<uint32_t*>(a.out + static_cast<size_t>(qrow[n]) * a.ldo + h * kHD +
                                             mt * 16 + hb * 8 + (lane & 3) * 2) = v;
            }
        }
      }
    }
    __syncthreads();  // buffer `buf` (halo + table) is rewritten by a later stage
    if (++js == nslots) {
      js = 0;
      ++hi;
    }
  }
}

// Per-shape launch policy: heads per CTA (their halos pipelined through
// two buffers) and double buffering. PSWA_ATTN_HPC / PSWA_ATTN_DBUF override
// for experiments. Context: 4 heads per CTA, double-buffered (measured with
// heavy-first tiles: 118 us per layer vs 125 with 2 heads, 140 with 1);
// steps: 1 head, single-buffered (13.2 us; double-buffered 18.0).
int env_int(const char* n, int dflt) {
  const char* e = std::getenv(n);
  return e ? std::atoi(e) : dflt;
}

int box_buf_bytes(int halo_keys) { return (halo_keys * 64 + 1023) / 1024 * 1024; }

int smem_bytes(int halo_keys, int dbuf, int qw) {
  // alignment slack + K/V buffers + 2 fp16 score-offset tables + barriers + band keys
  // (75.5 KB for a single-buffered 8-query step tile: 3 CTAs per SM)
  return 1024 + (dbuf ? 4 : 2) * box_buf_bytes(halo_keys) + 2 * kAttnMaxBandKeys * qw * 2 + 16 +
         kAttnMaxBandKeys * 2;
}

__global__ void score_table_kernel(const float* __restrict__ bias, int taps_total, const int8_t* __restrict__ taps,
                                   int n, int nsl, __half* __restrict__ out) {
  // out[h][k][i] = half(log2e * bias[h][k*49 + taps[i]]) or -inf (i < n = nbk*8)
  const int h = blockIdx.y, k = blockIdx.z;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int t = taps[i];
    out[(static_cast<size_t>(h) * nsl + k) * n + i] =
        __float2half_rn(t >= 0 ? bias[h * taps_total + k * 49 + t] * kLog2e : -INFINITY);
  }
}

template <int NP, int QW>
void launch_t8(const AttnArgs& a, const CUtensorMap& map, int halo_keys, int ntiles, int heads,
               int warps, cudaStream_t st) {
  launch_k(window_attn_t8_kernel<NP, QW>, dim3(heads / a.hpc, ntiles), dim3(warps * 32),
           smem_bytes(halo_keys, a.dbuf, QW), st, a, map);
}

}  // namespace

bool window_attention_tiles_supported(int hd, int win_h, int win_w) {
  return hd == kHD && win_h == 7 && win_w == 7;
}

int window_attention_tiles_smem(int halo_keys, bool) { return smem_bytes(halo_keys, 1, 16); }

void build_score_tables(const float* bias, int heads, int wt, AttnShape shape, __half* out,
                        cudaStream_t st) {
  const int nsl = wt > 0 ? wt : 1, n = shape.nbk * shape.qw;
  if (n == 0) return;
  score_table_kernel<<<dim3((n + 255) / 256, heads, nsl), 256, 0, st>>>(bias, nsl * 49, shape.taps, n,
                                                                       nsl, out);
  PSWA_LAUNCH_CHECK();
}

void window_attention_tiles_init(int max_smem_bytes) {
  PSWA_CUDA(cudaFuncSetAttribute(window_attn_t8_kernel<1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem_bytes));
  PSWA_CUDA(cudaFuncSetAttribute(window_attn_t8_kernel<2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem_bytes));
  PSWA_CUDA(cudaFuncSetAttribute(window_attn_t8_kernel<2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem_bytes));
}

void window_attention_tiles(const __half* q, int ldq, const int32_t* tiles, int ntiles,
                            int warps_per_tile, int halo_rows, int halo_width, AttnShape shape,
                            const CUtensorMap& kv_map, int heads, int wt, const __half* tables,
                            __half* out, int ldo, cudaStream_t st) {
  if (ntiles <= 0) return;
  if (shape.nbk % 16 || shape.nbk > kAttnMaxBandKeys) throw std::invalid_argument("attention shape");
  static const int hpc3 = env_int("PSWA_ATTN_HPC", 4), hpc2 = env_int("PSWA_ATTN_HPC2", 1);
  static const int dbuf3 = env_int("PSWA_ATTN_DBUF", 1), dbuf2 = env_int("PSWA_ATTN_DBUF2", 0);
  int hpc = wt > 0 ? hpc3 : hpc2;
  while (heads % hpc) --hpc;
  const int hk = halo_rows * halo_width;
  AttnArgs a{q, ldq, tiles, heads * kHD, wt, tables, wt > 0 ? wt : 1, out, ldo, shape, halo_width,
             box_buf_bytes(hk), wt > 0 ? dbuf3 : dbuf2, hpc};
  if (shape.qw == 16) {
    if (shape.nbk > 2 * 16 * pass_chunks<16>()) throw std::invalid_argument("attention shape (16 queries)");
    launch_t8<2, 16>(a, kv_map, hk, ntiles, heads, warps_per_tile, st);
  } else if (shape.nbk <= 16 * pass_chunks<8>()) {
    launch_t8<1, 8>(a, kv_map, hk, ntiles, heads, warps_per_tile, st);
  } else {
    launch_t8<2, 8>(a, kv_map, hk, ntiles, heads, warps_per_tile, st);
  }
  PSWA_LAUNCH_CHECK();
}

}  // namespace pswa_dev
