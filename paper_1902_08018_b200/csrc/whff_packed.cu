// whff_packed.cu -- kernels of the tile-packed layout (whff_packed.cuh):
// the fused decode + GEMV that reads it (k_pk_gemv2, TMA-staged: the
// coefficient evaluation -- the hot path -- and the exact evaluation with the
// reference's binary32 products), decode-only words and the exception side
// list, and their host launchers (whff_packed_api.h).  The packer is
// whff_pack.cu.
#include <cstddef>
#include <type_traits>

#include "whff_common.cuh"
#include "whff_packed.cuh"
#include "whff_packed_api.h"

// f(std::integral_constant<int, c>) for c = C0..C1, fully unrolled
template <int C0, int C1, class F>
__device__ __forceinline__ void unroll_range(F&& f) {
  if constexpr (C0 <= C1) {
    f(std::integral_constant<int, C0>());
    unroll_range<C0 + 1, C1>(f);
  }
}

// field widths / layout of a segment header
__device__ __forceinline__ void seg_layout(const pk::Seg& S, int W[16], pk::Layout& f) {
#pragma unroll
  for (int c = 0; c < 16; ++c) W[c] = pk::seg_W(S, c);
  pk::make_layout(pk::seg_We(S), W, f);
}

// The first kFastWords words of the record of (row i, lane) of a tile in
// global memory (words past the record read as 0).
__device__ __forceinline__ void pk_rec_fast(uint32_t a[pk::kFastWords], const uint32_t* tile, int R, int lane,
                                            int i) {
#pragma unroll
  for (int k = 0; k < pk::kFastWords; ++k) a[k] = k < R ? ldg(tile + pk::tile_word(k, lane, i)) : 0u;
}

// one field's parameters from the warp's shared table, loaded where used (a
// volatile load: ptxas would otherwise hoist all sixteen 16-byte loads to
// the top of the tile and spend 64 registers on them)
__device__ __forceinline__ pk::FieldPar lds_par(const pk::FieldPar* p) {
  pk::FieldPar r;
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}

// All 16 coefficients (sequency order) of one fast-path record (decode-only
// and exact evaluation; the pair of each group is selected per segment).
template <bool HASA = true, bool HASB = true>
__device__ __forceinline__ void pk_fields_int(const uint32_t a[pk::kFastWords], const pk::FieldPar* par /* smem */,
                                              bool k2, bool kA, bool kB, int32_t q[16]) {
  q[0] = pk::field_dc(a[0], a[1], lds_par(par));
  q[1] = pk::field_i(a[0], a[1], lds_par(par + 1));
  q[2] = pk::field_i(k2 ? a[1] : a[0], k2 ? a[2] : a[1], lds_par(par + 2));
  const uint32_t hA = kA ? a[2] : a[1], lA = kA ? a[3] : a[2];
  const uint32_t hB = kB ? a[3] : a[2], lB = kB ? a[4] : a[3];
#pragma unroll
  for (int c = 3; c <= 8; ++c) q[c] = HASA ? pk::field_i(hA, lA, lds_par(par + c)) : 0;
#pragma unroll
  for (int c = 9; c < 16; ++c) q[c] = HASB ? pk::field_i(hB, lB, lds_par(par + c)) : 0;
}

// Generic path: the whole record (any L) of (row i, lane) into rec[].
__device__ __noinline__ void pk_generic_record(const uint32_t* tile, int R, int lane, int i, uint32_t* rec) {
  for (int k = 0; k <= pk::kMaxRecordWords; ++k) rec[k] = k < R ? ldg(tile + pk::tile_word(k, lane, i)) : 0u;
}

// Generic segments (fields wider than the fast path allows, L up to 457):
// one record parsed sequentially; out of line, results through memory.
__device__ __noinline__ void pk_generic_parse(const pk::Seg* Sp, const uint32_t* tile, int lane, int i, int32_t* q,
                                              uint32_t* ed) {
  const pk::Seg S = *Sp;
  int W[16];
  pk::Layout f;
  seg_layout(S, W, f);
  uint32_t rec[pk::kMaxRecordWords + 1];
  pk_generic_record(tile, pk::rec_words(f.L), lane, i, rec);
  pk::parse_record(f, W, rec, *ed, q);
}

template <int POL>
struct PkAcc {
  using T = typename std::conditional<POL == WHFF_POLICY_SINGLE, float, double>::type;
  T v[4][4];
};

// Exceptions of a segment: the warp adds their exact spatial products
// (binary32 words x v; policy products) into the warp's per-row sums r[16]
// (shared memory): lanes 0..15 take the block's 16 words, row sums as
// (p0 + p1) + (p2 + p3), exceptions in list order.
template <int POL, typename T>
__device__ __forceinline__ void pk_exceptions(const PkView& P, const float* v, uint64_t band,
                                              uint32_t e0, uint32_t ne, int lane, T* rs) {
  for (uint32_t e = e0; e < e0 + ne; ++e) {
    T p = (T)0;
    int i = 0;
    if (lane < 16) {
      const uint64_t b = P.exc_block[e];
      const uint64_t brow = b / P.g.bc, bcol = b % P.g.bc;
      i = (int)(brow - band * pk::kBand);
      const uint64_t col = bcol * 4 + (lane & 3);
      float x = __uint_as_float(P.exc_words[16 * (uint64_t)e + lane]);
      float vj = 0.0f;
      if (col < P.g.cols) vj = ldg(v + col);
      else x = 0.0f;
      if (POL == WHFF_POLICY_DOUBLE) p = (T)__dmul_rn((double)x, (double)vj);
      else p = (T)__fmul_rn(x, vj);
    }
    p = p + __shfl_xor_sync(0xFFFFFFFFu, p, 1);
    p = p + __shfl_xor_sync(0xFFFFFFFFu, p, 2);
    if (lane < 16 && (lane & 3) == 0) rs[4 * i + (lane >> 2)] = rs[4 * i + (lane >> 2)] + p;
    __syncwarp();
  }
}

// acc[r] += product row r of words x with v (the policy's arithmetic,
// columns in order: the reference's sequential row order within a block)
template <int POL, typename AT>
__device__ __forceinline__ void pk_acc_words(AT acc[4], const float x[16], const float vv[4]) {
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float xv = x[4 * r + j];
      if (POL == WHFF_POLICY_MIXED) acc[r] = __dadd_rn(acc[r], (double)__fmul_rn(xv, vv[j]));
      else if (POL == WHFF_POLICY_SINGLE) acc[r] = __fadd_rn(acc[r], __fmul_rn(xv, vv[j]));
      else acc[r] = __dadd_rn(acc[r], __dmul_rn((double)xv, (double)vv[j]));
    }
}

// the job (stream, vector, output, rows) of a global band and its first band
__device__ __forceinline__ const PkJob& pk_job(const PkTable& T, uint64_t gband, uint64_t& first) {
  first = 0;
  if (T.jobs == nullptr) return T.single;
  int lo = 0, hi = T.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (T.prefix[mid] <= gband) lo = mid; else hi = mid - 1;
  }
  first = T.prefix[lo];
  return T.jobs[lo];
}

// Each of a band's kVW virtual warps publishes its partial record (the
// per-row sums of its segments, and of its exceptions); k_pk_combine then
// combines them with a fixed butterfly per row -- the same bits whatever
// launch (single call, row range, field plan) computes the band -- and
// coefficient evaluation applies the inverse lift G once per block-row.  The
// combine is a second kernel (the launch boundary orders the records): the
// main kernel has no atomics and no memory fences.
template <int POL, typename AT>
__device__ __forceinline__ void pk_store_partial(const PkTable& T, uint64_t gband, int vw, int lane,
                                                 const AT* dsum /* [16] per lane: row 4i+r */, bool dsum_lane_major,
                                                 const AT* rs) {
  PkRec* grec = T.recs + gband * kVW;
  if (dsum_lane_major) {
    // dsum[0] of lane 2m holds row m (the transpose reduction of k_pk_gemv2)
    if ((lane & 1) == 0) {
      if (POL == WHFF_POLICY_SINGLE) grec[vw].f[lane >> 1] = (float)dsum[0];
      else grec[vw].d[lane >> 1] = (double)dsum[0];
    }
    if (lane < 16) {
      if (POL == WHFF_POLICY_SINGLE) grec[vw].rf[lane] = (float)rs[lane];
      else grec[vw].r[lane] = (double)rs[lane];
    }
  } else if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (POL == WHFF_POLICY_SINGLE) {
        grec[vw].f[k] = (float)dsum[k];
        grec[vw].rf[k] = (float)rs[k];
      } else {
        grec[vw].d[k] = (double)dsum[k];
        grec[vw].r[k] = (double)rs[k];
      }
    }
  }
}

template <int EVAL, int POL, typename AT>
__device__ __forceinline__ void pk_combine_band(const PkJob& J, const PkView& P, const PkRec* grec, uint64_t band,
                                                int nrows, int lane, unsigned long long* status) {
  // lane = value (0..15: the block sums D of row lane, 16..31: the exception
  // sums R of row lane - 16), read from the 32 records (coalesced: one
  // 128-byte line per record and kind), then summed over the records in the
  // fixed xor-butterfly order (16, 8, 4, 2, 1) -- the pairwise tree that
  // leaves the same bits in every lane of a shuffle butterfly.
  AT x[kVW];
#pragma unroll
  for (int w = 0; w < kVW; ++w) {
    if (POL == WHFF_POLICY_SINGLE) x[w] = (AT)__ldcg(lane < 16 ? &grec[w].f[lane] : &grec[w].rf[lane - 16]);
    else x[w] = (AT)__ldcg(lane < 16 ? &grec[w].d[lane] : &grec[w].r[lane - 16]);
  }
#pragma unroll
  for (int o = kVW / 2; o > 0; o >>= 1)
#pragma unroll
    for (int w = 0; w < o; ++w) x[w] = x[w] + x[w + o];
  const AT tot = x[0];
  // row m = lane (< 16) of the band: its R and the D of the block-row's 4 rows
  const int i = (lane >> 2) & 3, rr = lane & 3;
  const AT rsel = __shfl_sync(0xFFFFFFFFu, tot, 16 + (lane & 15));
  const AT d0 = __shfl_sync(0xFFFFFFFFu, tot, 4 * i + 0), d1 = __shfl_sync(0xFFFFFFFFu, tot, 4 * i + 1);
  const AT d2 = __shfl_sync(0xFFFFFFFFu, tot, 4 * i + 2), d3 = __shfl_sync(0xFFFFFFFFu, tot, 4 * i + 3);
  if (lane < 16) {
    const uint64_t row = (band * pk::kBand + i) * 4 + rr;
    if (i < nrows && row >= J.row_begin && row < J.row_end && row < P.g.rows) {
      float out;
      if (EVAL == WHFF_EVAL_COEFF) {
        const AT dd[4] = {d0, d1, d2, d3};
        if (POL == WHFF_POLICY_SINGLE) {
          float t = (float)rsel;
#pragma unroll
          for (int a = 0; a < 4; ++a) t = __fmaf_rn(c_G[rr][a], (float)dd[a], t);
          out = t;
        } else {
          double t = (double)rsel;
#pragma unroll
          for (int a = 0; a < 4; ++a) t = __fma_rn((double)c_G[rr][a], (double)dd[a], t);
          out = __double2float_rn(t);
        }
      } else {
        if (POL == WHFF_POLICY_SINGLE) out = __fadd_rn((float)tot, (float)rsel);
        else out = __double2float_rn(__dadd_rn((double)tot, (double)rsel));
      }
      J.y[row - J.row_begin] = out;
      if (!isfinite(out)) atomicMin(status, (unsigned long long)row);
    }
  }
}

// ---------------------------------------------------------------------------
// fused decode + GEMV, TMA-staged (the hot path)
// ---------------------------------------------------------------------------
// 8 CTAs of 4 warps per band; the band's 32 virtual warps each take segments
// vw, vw + 32, ... .  Built for the B200's issue rate:
//   * every warp runs its own kP2Stages-deep ring of shared-memory stages;
//     one elected lane fills each stage with two 1-D bulk copies
//     (cp.async.bulk, the TMA engine): up to p2_item_tiles(R) consecutive
//     tiles of a segment (4 block-rows x 32 block-columns of records each,
//     word-major, contiguous in HBM) and their slice of U = G^T v, completing on the stage's
//     mbarrier: no registers hold loads in flight and the copies of the next
//     items overlap the decode of this one;
//   * one 16-byte shared load per record word gives that word of all four
//     block-rows; the rows are decoded as two pairs with the packed-f32x2
//     pipe (FFMA2/FADD2 for the exact conversions, FFMA2 for coefficient x u
//     and for the 2^k-scaled accumulation); the small fields of a group (c =
//     3..8, 9..15) come out of one 64-bit shift per row and one LOP3 each;
//   * the per-segment field parameters are precomputed by the packer and
//     prefetched one segment ahead; the tile body is compiled for the two
//     layouts almost every smooth segment has (all groups present, or DC and
//     the two large AC coefficients only) besides the general one;
//   * per segment (8 tiles) each lane sums its 2^k (Q u) terms per (block-
//     row, row) in binary32; at the segment's end the warp reduces the 16
//     sums over its 32 lanes with a transpose reduction (the first stage in
//     binary32, the rest in binary64), after which lane 2m holds row m -- one
//     binary64 accumulator per lane, no per-block conversions.
// Generic segments (fields too wide for the fast path) and exceptions take
// per-lane paths on global memory.
#ifndef WHFF_P2_STAGES
#define WHFF_P2_STAGES 2
#endif
#ifndef WHFF_P2_MINB
#define WHFF_P2_MINB 4
#endif
constexpr int kP2Warps = 4;                              // warps per CTA
constexpr int kP2Split = kPkVW / kP2Warps;               // CTAs per band
constexpr int kP2Stages = WHFF_P2_STAGES;
// A stage holds the next t tiles of one segment: their records (R words per
// lane and block-row: R x 512 bytes per tile, contiguous in HBM) followed by
// their slices of U (512 bytes per tile), t = 12 / (R + 1) capped at a
// segment -- 2 tiles at R = 4, 5; 3 at R = 3 (most FixedRate(8) segments); 4
// at R = 2 (FixedAccuracy); 6 at R = 1 -- so the per-item costs (barrier
// wait, copy issue, cursor) are spread over as many blocks as 6 KB allows.
#ifndef WHFF_P2_UNITS
#define WHFF_P2_UNITS 12
#endif
constexpr int kP2StageUnits = WHFF_P2_UNITS;
constexpr int kP2StageBytes = kP2StageUnits * 512;
// (a nibble table: min(8, units / (R + 1)) for the fast path's R = 1..5, no division)
constexpr uint32_t p2_item_table(int units) {
  uint32_t t = 0;
  for (int R = 1; R <= 5; ++R) {
    const int n = units / (R + 1) < pk::kSegTiles ? units / (R + 1) : pk::kSegTiles;
    t |= (uint32_t)n << (4 * (R - 1));
  }
  return t;
}
constexpr uint32_t kP2ItemTable = p2_item_table(kP2StageUnits);
static_assert(pk::kFastWords == 5 && kP2StageUnits >= 6, "every fast-path record fits one tile per stage");
__device__ __forceinline__ int p2_item_tiles(int R) { return (int)((kP2ItemTable >> (4 * (R - 1))) & 15u); }
constexpr int kP2HdrRing = 16;                           // segment headers held per warp
constexpr int kP2HdrChunk = 8;

// Per-warp state the tile loop does not touch lives in shared memory (read
// and written through volatile accesses), so it holds no registers across
// the decode: the job's pointers, the producer's cursor, the header ring fill.
struct alignas(16) P2Ctl {
  uint64_t pbody, usrc;                  // next item: body and U source addresses
  uint32_t pk, pt, pntl, pslot;          // producer cursor: segment, tile, its tiles, stage
  uint32_t ptw, nseg, hdr_loaded, ntile; // words per tile of segment pk; warp constants
  uint32_t hdr_landed, segt, pad1, pad2;  // header ring: slots known to have landed; tiles per segment
  uint64_t body, U, gsegs, gpars, policy, pad;
};
template <typename AT>
struct alignas(128) P2Warp {
  uint8_t stage[kP2Stages][kP2StageBytes];
  uint64_t bar[kP2Stages];
  pk::Seg seg[kP2HdrRing];     // the producer's header ring
  pk::Seg cur[2];              // the consumer's: this segment's and the next one's (cp.async prefetch)
  pk::FieldPar par[2][16];     // this segment's and the next one's (cp.async prefetch)
  AT rs[16];
  P2Ctl ctl;
};
__device__ __forceinline__ uint32_t ctl_ld32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t ctl_ld64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 ctl_ld128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void ctl_st128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint64_t u64_of(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }
__device__ __forceinline__ void ctl_st32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void ctl_st64(uint32_t a, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ pk::FieldPar lds_par_a(uint32_t a) {
  pk::FieldPar r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}

// The transpose reduction of a segment's 16 per-lane sums over the warp, in
// binary32: afterwards lane l holds the sum over the 32 lanes of row m = l >> 1
// of the band (m = 4 i + r), converted to AT once.  Each stage (xor 16, 8, 4,
// 2) halves the values a lane keeps -- the butterfly restricted to them --
// on row pairs with FADD2 while there are pairs; xor 1 finishes.
template <typename AT>
__device__ __forceinline__ AT seg_reduce(const float2 s[2][4], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  float2 d[4];   // d[j] = rows (j, 4 + j) of the kept block-row pair: m - 8 b4 = 4 i' + r
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const float2 send = b4 ? s[0][r] : s[1][r];
    const float2 mine = b4 ? s[1][r] : s[0][r];
    d[r] = __fadd2_rn(mine, make_float2(__shfl_xor_sync(0xFFFFFFFFu, send.x, 16),
                                        __shfl_xor_sync(0xFFFFFFFFu, send.y, 16)));
  }
  // xor 8: keep i' = b3 (values 4 i' + r, r = 0..3) -> f = rows r = 0..3
  float2 f[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    // (value 2j, value 2j+1) of i' = 0 are d[2j].x, d[2j+1].x; of i' = 1: .y
    const float2 lo = make_float2(d[2 * j].x, d[2 * j + 1].x), hi = make_float2(d[2 * j].y, d[2 * j + 1].y);
    const float2 send = b3 ? lo : hi;
    const float2 mine = b3 ? hi : lo;
    f[j] = __fadd2_rn(mine, make_float2(__shfl_xor_sync(0xFFFFFFFFu, send.x, 8),
                                        __shfl_xor_sync(0xFFFFFFFFu, send.y, 8)));
  }
  // xor 4: keep r in {2 b2, 2 b2 + 1}
  const float2 send4 = b2 ? f[0] : f[1];
  const float2 mine4 = b2 ? f[1] : f[0];
  const float2 g = __fadd2_rn(mine4, make_float2(__shfl_xor_sync(0xFFFFFFFFu, send4.x, 4),
                                                 __shfl_xor_sync(0xFFFFFFFFu, send4.y, 4)));
  // xor 2: keep r = 2 b2 + b1
  const float send2 = b1 ? g.x : g.y;
  const float mine2 = b1 ? g.y : g.x;
  const float h = mine2 + __shfl_xor_sync(0xFFFFFFFFu, send2, 2);
  return (AT)(h + __shfl_xor_sync(0xFFFFFFFFu, h, 1));
}

// tile-body specialisations (per segment): every group present on its first
// candidate pair, groups on the group path (the common rate layout); the same
// without group B (c = 9..15 all zero: the next most common rate layout); DC
// and c = 1, 2 only (the common precision / accuracy layout); anything else
enum { kSpecFull = 0, kSpecDC = 1, kSpecAny = 2, kSpecFullA = 3 };

// One tile of a fast segment from shared memory: adds 2^k (Q u) of the
// lane's block in each of the four block-rows to s[h][r].
// tw: the stage address of the lane's first record word (16 * lane added);
// uw: the stage address of the lane's U entry; par: the warp's parameters.
template <int SPEC>
__device__ __forceinline__ void p2_tile(uint32_t tw, uint32_t uw, uint32_t par, bool m12, bool k2, bool hasA,
                                        bool gA, bool kA, bool hasB, bool gB, bool kB, int We, uint32_t ebase_bits,
                                        float2 s[2][4]) {
  constexpr int NW = SPEC == kSpecDC ? 2 : SPEC == kSpecFull ? 4 : SPEC == kSpecFullA ? 3 : pk::kFastWords;
  float u[4];
  {
    uint4 t;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "r"(uw));
    u[0] = __uint_as_float(t.x);
    u[1] = __uint_as_float(t.y);
    u[2] = __uint_as_float(t.z);
    u[3] = __uint_as_float(t.w);
  }
  // a[i][k]: word k of block-row i's record (one 16-byte load per word;
  // words past the record are stale and only ever shifted out)
  uint32_t a[4][pk::kFastWords];
#pragma unroll
  for (int kw = 0; kw < pk::kFastWords; ++kw) {
    if (kw < NW) {
      uint4 t;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "r"(tw + 512 * kw));
      a[0][kw] = t.x;
      a[1][kw] = t.y;
      a[2][kw] = t.z;
      a[3][kw] = t.w;
    } else {
      a[0][kw] = a[1][kw] = a[2][kw] = a[3][kw] = 0u;
    }
  }
  // w[h][r] = (w of block-row 2h, of block-row 2h + 1), row r
  float2 w[2][4];
  {
    const pk::FieldPar p0 = lds_par_a(par);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float f0a = __int2float_rn(pk::field_dc(a[2 * h][0], a[2 * h][1], p0));
      const float f0b = __int2float_rn(pk::field_dc(a[2 * h + 1][0], a[2 * h + 1][1], p0));
      w[h][0] = __fmul2_rn(make_float2(f0a, f0b), make_float2(u[0], u[0]));
      w[h][1] = w[h][2] = w[h][3] = make_float2(0.0f, 0.0f);
    }
  }
  // kSpecAny: the pair of a group chosen per segment, selected into b[][]
  uint32_t b[4][2];
  // the pair (hi, lo) of row i for a field: a[i][kk], a[i][kk + 1], or b[i][]
  auto hi = [&](auto K, auto B, int i) -> uint32_t {
    if constexpr (decltype(B)::value) return b[i][0];
    else return a[i][decltype(K)::value];
  };
  auto lo = [&](auto K, auto B, int i) -> uint32_t {
    if constexpr (decltype(B)::value) return b[i][1];
    else return a[i][decltype(K)::value + 1];
  };
  // Each field's parameters are loaded (shared memory, volatile) one field
  // ahead of its use so the load latency hides behind the previous field.
  // c = 1, 2: integer fields (up to 28 bits), binary32 by rounding
  auto field_int = [&](auto C, auto K, auto B, const pk::FieldPar& p) {
    constexpr int c = decltype(C)::value;
    constexpr int r = seq_pos(c) >> 2, j = seq_pos(c) & 3;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float2 q = make_float2(__int2float_rn(pk::field_i(hi(K, B, 2 * h), lo(K, B, 2 * h), p)),
                                   __int2float_rn(pk::field_i(hi(K, B, 2 * h + 1), lo(K, B, 2 * h + 1), p)));
      w[h][r] = __ffma2_rn(q, make_float2(u[j], u[j]), w[h][r]);
    }
  };
  // c >= 3, field path: two funnel shifts put the field under the binary32
  // exponent of 2^23, FADD2 removes 2^23 + 2^(W-1): exact
  auto field = [&](auto C, auto K, auto B, const pk::FieldPar& p) {
    constexpr int c = decltype(C)::value;
    constexpr int r = seq_pos(c) >> 2, j = seq_pos(c) & 3;
    const float off = __uint_as_float(p.w);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t fa = fsr(pk::fsl64(hi(K, B, 2 * h), lo(K, B, 2 * h), p.x), p.y, p.z);
      const uint32_t fb = fsr(pk::fsl64(hi(K, B, 2 * h + 1), lo(K, B, 2 * h + 1), p.x), p.y, p.z);
      const float2 q = __fadd2_rn(make_float2(__uint_as_float(fa), __uint_as_float(fb)), make_float2(off, off));
      w[h][r] = __ffma2_rn(q, make_float2(u[j], u[j]), w[h][r]);
    }
  };
  // c >= 3, group path: the group's bits at the bottom of a register (one
  // 64-bit shift per row), one LOP3 per field, one FFMA2 converts two rows
  struct X4 {
    uint32_t v0, v1, v2, v3;
  };
  auto fieldg = [&](auto C, const X4& x, const pk::FieldPar& p) {
    constexpr int c = decltype(C)::value;
    constexpr int r = seq_pos(c) >> 2, j = seq_pos(c) & 3;
    const float sc2 = __uint_as_float(p.y), off = __uint_as_float(p.z);
    const uint32_t f0 = (x.v0 & p.x) | pk::kMagic, f1 = (x.v1 & p.x) | pk::kMagic;
    const uint32_t f2 = (x.v2 & p.x) | pk::kMagic, f3 = (x.v3 & p.x) | pk::kMagic;
    const float2 q0 = __ffma2_rn(make_float2(__uint_as_float(f0), __uint_as_float(f1)), make_float2(sc2, sc2),
                                 make_float2(off, off));
    const float2 q1 = __ffma2_rn(make_float2(__uint_as_float(f2), __uint_as_float(f3)), make_float2(sc2, sc2),
                                 make_float2(off, off));
    w[0][r] = __ffma2_rn(q0, make_float2(u[j], u[j]), w[0][r]);
    w[1][r] = __ffma2_rn(q1, make_float2(u[j], u[j]), w[1][r]);
  };
  // fields c0..c1 in order, parameters one field ahead; G: group path; M:
  // c = 1, 2 in the magic-number format (seg_m12)
  auto run = [&](auto C0, auto C1, auto K, auto B, auto G, auto M) {
    constexpr int c0 = decltype(C0)::value, c1 = decltype(C1)::value;
    constexpr bool grp = decltype(G)::value;
    pk::FieldPar p = lds_par_a(par + 16 * c0);
    X4 x{};
    if constexpr (grp) {
      x.v0 = pk::group_bits(hi(K, B, 0), lo(K, B, 0), p.w);
      x.v1 = pk::group_bits(hi(K, B, 1), lo(K, B, 1), p.w);
      x.v2 = pk::group_bits(hi(K, B, 2), lo(K, B, 2), p.w);
      x.v3 = pk::group_bits(hi(K, B, 3), lo(K, B, 3), p.w);
    }
    unroll_range<c0, c1>([&](auto CC) {
      constexpr int c = decltype(CC)::value;
      pk::FieldPar pn = p;
      if constexpr (c < c1) pn = lds_par_a(par + 16 * (c + 1));
      if constexpr (grp) fieldg(CC, x, p);
      else if constexpr (c <= 2 && !decltype(M)::value) field_int(CC, K, B, p);
      else field(CC, K, B, p);
      p = pn;
    });
  };
  // b[i][] = pair kk (up: kk + 1) of row i
  auto pick = [&](auto K, bool up) {
    constexpr int kk = decltype(K)::value;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      b[i][0] = up ? a[i][kk + 1] : a[i][kk];
      b[i][1] = up ? a[i][kk + 2] : a[i][kk + 1];
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  using T_ = std::true_type;
  using F_ = std::false_type;
  using C1_ = std::integral_constant<int, 1>;
  using C2_ = std::integral_constant<int, 2>;
  using C3_ = std::integral_constant<int, 3>;
  using C8_ = std::integral_constant<int, 8>;
  using C9_ = std::integral_constant<int, 9>;
  using C15_ = std::integral_constant<int, 15>;
  if (SPEC != kSpecAny) {
    run(C1_(), C2_(), I0(), F_(), F_(), T_());
    if (SPEC == kSpecFull || SPEC == kSpecFullA) run(C3_(), C8_(), I1(), F_(), T_(), F_());
    if (SPEC == kSpecFull) run(C9_(), C15_(), I2(), F_(), T_(), F_());
  } else {
    if (m12) run(C1_(), C1_(), I0(), F_(), F_(), T_());
    else run(C1_(), C1_(), I0(), F_(), F_(), F_());
    pick(I0(), k2);
    if (m12) run(C2_(), C2_(), I0(), T_(), F_(), T_());
    else run(C2_(), C2_(), I0(), T_(), F_(), F_());
    if (hasA) {
      pick(I1(), kA);
      if (gA) run(C3_(), C8_(), I1(), T_(), T_(), F_());
      else run(C3_(), C8_(), I1(), T_(), F_(), F_());
    }
    if (hasB) {
      pick(I2(), kB);
      if (gB) run(C9_(), C15_(), I2(), T_(), T_(), F_());
      else run(C9_(), C15_(), I2(), T_(), F_(), F_());
    }
  }
  // s += w 2^k: the product is exact, one rounding per term (most segments
  // have a single emax, W_e = 0: one scale for the whole tile)
  if (We == 0) {
    const float sc = __uint_as_float(ebase_bits);
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int r = 0; r < 4; ++r) s[h][r] = __ffma2_rn(w[h][r], make_float2(sc, sc), s[h][r]);
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t ea = pk::field_edelta(a[2 * h][0], We), eb = pk::field_edelta(a[2 * h + 1][0], We);
      const float2 sc =
          make_float2(__uint_as_float(ebase_bits + (ea << 23)), __uint_as_float(ebase_bits + (eb << 23)));
#pragma unroll
      for (int r = 0; r < 4; ++r) s[h][r] = __ffma2_rn(w[h][r], sc, s[h][r]);
    }
  }
}

// The transpose reduction of 16 per-lane AT values (m = 4 i + r) over the
// warp, every stage in AT: afterwards lane l holds row m = l >> 1.
template <typename AT>
__device__ __forceinline__ AT seg_reduce16(const AT d[16], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  AT e[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const AT send = b4 ? d[j] : d[8 + j];
    const AT mine = b4 ? d[8 + j] : d[j];
    e[j] = mine + __shfl_xor_sync(0xFFFFFFFFu, send, 16);
  }
  AT f[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const AT send = b3 ? e[j] : e[4 + j];
    const AT mine = b3 ? e[4 + j] : e[j];
    f[j] = mine + __shfl_xor_sync(0xFFFFFFFFu, send, 8);
  }
  AT g[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const AT send = b2 ? f[j] : f[2 + j];
    const AT mine = b2 ? f[2 + j] : f[j];
    g[j] = mine + __shfl_xor_sync(0xFFFFFFFFu, send, 4);
  }
  const AT send = b1 ? g[0] : g[1];
  const AT mine = b1 ? g[1] : g[0];
  AT h = mine + __shfl_xor_sync(0xFFFFFFFFu, send, 2);
  return h + __shfl_xor_sync(0xFFFFFFFFu, h, 1);
}

// Exact evaluation, one tile from shared memory: the four block-rows'
// binary32 words, bit-exact with codec.decompress (int32 lift, exact
// dequantisation, codec.py:128-218), times v in the policy's arithmetic,
// added to se[4 i + r] in (row, column) order.
// tw: stage address of the lane's first record word; vwa: of its v entry.
// HASA / HASB: coefficient groups 3..8 / 9..15 present in the segment (an
// absent group is all zeros: its fields are not read and the lift folds them).
template <int POL, typename AT, bool HASA, bool HASB>
__device__ __forceinline__ void p2_tile_exact(uint32_t tw, uint32_t vwa, const pk::FieldPar* par, bool k2, bool kA,
                                              bool kB, int We, uint32_t ebase, AT se[16]) {
  float v[4];
  {
    uint4 t;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w) : "r"(vwa));
    v[0] = __uint_as_float(t.x);
    v[1] = __uint_as_float(t.y);
    v[2] = __uint_as_float(t.z);
    v[3] = __uint_as_float(t.w);
  }
  // The four block-rows, one loop trip each (not unrolled: the body is
  // long).  se[] is indexed statically: each trip works on se[0..3] and
  // rotates the array by one block-row, so after four trips every sum is
  // back in place (a dynamic index would put se[] in local memory).
#if WHFF_EXACT_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int i = 0; i < 4; ++i) {
    uint32_t a[pk::kFastWords];
#pragma unroll
    for (int kw = 0; kw < pk::kFastWords; ++kw)
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a[kw]) : "r"(tw + 512 * kw + 4 * i));
    int32_t q[16], t[16];
    pk_fields_int<HASA, HASB>(a, par, k2, kA, kB, q);
    lift_signed(q, t);
    // dequantisation (codec.py:201-206) on the packed pipe when the scale
    // is a normal-or-subnormal binary32 power of two (single rounding,
    // as dequant_words); otherwise the binary64 path
    const uint32_t emax = ebase + pk::field_edelta(a[0], We);
    const int k = (int)emax - kEmaxBias - kQuantBits;
    float x[16];
    if (emax != 0u && dequant_fast_ok(k)) {
      const float s = scale_f32(k);
#pragma unroll
      for (int m = 0; m < 16; m += 2) {
        const float2 w = __fmul2_rn(make_float2((float)t[m], (float)t[m + 1]), make_float2(s, s));
        x[m] = w.x;
        x[m + 1] = w.y;
      }
    } else {
      dequant_words(t, emax, x);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      AT acc = se[r];
      if (POL == WHFF_POLICY_DOUBLE) {
#pragma unroll
        for (int j = 0; j < 4; ++j) acc = __dadd_rn(acc, __dmul_rn((double)x[4 * r + j], (double)v[j]));
      } else {
        // binary32 products two at a time, added in column order
#pragma unroll
        for (int j = 0; j < 4; j += 2) {
          const float2 p = __fmul2_rn(make_float2(x[4 * r + j], x[4 * r + j + 1]), make_float2(v[j], v[j + 1]));
          if (POL == WHFF_POLICY_MIXED) {
            acc = __dadd_rn(acc, (double)p.x);
            acc = __dadd_rn(acc, (double)p.y);
          } else {
            acc = __fadd_rn(acc, p.x);
            acc = __fadd_rn(acc, p.y);
          }
        }
      }
      se[r] = acc;
    }
    AT rot[16];   // rotate by one block-row (a register permutation)
#pragma unroll
    for (int m = 0; m < 16; ++m) rot[m] = se[(m + 4) & 15];
#pragma unroll
    for (int m = 0; m < 16; ++m) se[m] = rot[m];
  }
}

template <int EVAL, int POL>
__global__ void __launch_bounds__(32 * kP2Warps, WHFF_P2_MINB) k_pk_gemv2(PkTable T, unsigned long long* status) {
  using AT = typename PkAcc<POL>::T;
  constexpr bool kCoef = EVAL == WHFF_EVAL_COEFF;
  extern __shared__ __align__(128) uint8_t p2_smem[];
  const uint64_t gband = blockIdx.x / kP2Split;
  const int part = (int)(blockIdx.x % kP2Split);
  if (gband >= T.total_bands) return;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  P2Warp<AT>& W = reinterpret_cast<P2Warp<AT>*>(p2_smem)[warp];
  uint64_t first;
  const PkJob& J = pk_job(T, gband, first);
  const uint64_t band = J.band0 + (gband - first);
  const int vw = part * kP2Warps + warp;

  // shared-memory addresses (32-bit) of the warp's stages, barriers,
  // parameters and control block
  const uint32_t st0 = smem_addr(&W.stage[0][0]);
  const uint32_t bar0 = smem_addr(&W.bar[0]);
  const uint32_t par0 = smem_addr(&W.par[0][0]);
  const uint32_t ctl = smem_addr(&W.ctl);
  const uint32_t c_body = ctl + offsetof(P2Ctl, body), c_U = ctl + offsetof(P2Ctl, U);
  const uint32_t c_gsegs = ctl + offsetof(P2Ctl, gsegs), c_gpars = ctl + offsetof(P2Ctl, gpars);
  const uint32_t c_policy = ctl + offsetof(P2Ctl, policy), c_A = ctl + offsetof(P2Ctl, pbody);
  const uint32_t c_B = ctl + offsetof(P2Ctl, pk), c_C = ctl + offsetof(P2Ctl, ptw);
  const uint32_t c_pk = ctl + offsetof(P2Ctl, pk), c_pt = ctl + offsetof(P2Ctl, pt);
  const uint32_t c_pslot = ctl + offsetof(P2Ctl, pslot), c_pntl = ctl + offsetof(P2Ctl, pntl);
  const uint32_t c_nseg = ctl + offsetof(P2Ctl, nseg), c_hdr = ctl + offsetof(P2Ctl, hdr_loaded);
  const uint32_t c_ntile = ctl + offsetof(P2Ctl, ntile), c_landed = ctl + offsetof(P2Ctl, hdr_landed);
  const uint32_t c_segt = ctl + offsetof(P2Ctl, segt);
  {
    const PkView& P = J.p;
    const uint64_t nsegb = P.g.nsegb;
    const int nseg = nsegb > (uint64_t)vw ? (int)((nsegb - 1 - vw) / kVW + 1) : 0;
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      ctl_st64(c_body, reinterpret_cast<uint64_t>(P.body));
      ctl_st64(c_U, reinterpret_cast<uint64_t>(J.U));
      ctl_st64(c_gsegs, reinterpret_cast<uint64_t>(P.segs + band * nsegb + vw));
      ctl_st64(c_gpars, reinterpret_cast<uint64_t>(P.pars + (band * nsegb + vw) * 16));
      ctl_st64(c_policy, policy);
      ctl_st32(c_pk, 0);
      ctl_st32(c_pt, 0);
      ctl_st32(c_pslot, 0);
      ctl_st32(c_nseg, (uint32_t)nseg);
      ctl_st32(c_hdr, 0);
      ctl_st32(c_landed, 0);
      ctl_st32(c_segt, (uint32_t)P.g.segt);
      ctl_st32(c_ntile, (uint32_t)P.g.ntile);
    }
    if (lane < 16) W.rs[lane] = (AT)0;
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < kP2Stages; ++i) mbar_init(&W.bar[i], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }

  // Segment headers.  The producer walks them forward through a
  // shared-memory ring, kP2HdrChunk at a time; only it reads the ring, so a
  // chunk may overwrite any slot behind its cursor (however many generic
  // segments it skips).  Each chunk is copied with cp.async; when the
  // producer enters chunk c it also starts chunk c + 1, which it then finds
  // landed (a cp.async.wait_group makes sure).  The consumer reads its own
  // copy of each header (W.cur), prefetched one segment ahead like the
  // parameters.
  static_assert(kP2HdrRing == 2 * kP2HdrChunk, "the header ring holds two chunks");
  auto hdr_chunk = [&](int c) {   // cp.async chunk c into the ring (lanes 0..23: 3 x 16 bytes each)
    const int nseg = (int)ctl_ld32(c_nseg);
    const int kk = c * kP2HdrChunk + lane / 3;
    if (lane < 3 * kP2HdrChunk && kk < nseg) {
      const char* g = reinterpret_cast<const char*>(reinterpret_cast<const pk::Seg*>(ctl_ld64(c_gsegs)) +
                                                    (uint64_t)kVW * kk) + 16 * (lane % 3);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                   ::"r"(smem_addr(&W.seg[kk & (kP2HdrRing - 1)]) + 16 * (lane % 3)), "l"(g) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto ensure_hdr = [&](int k) {
    if (k < (int)ctl_ld32(c_landed)) return;
    int loaded = (int)ctl_ld32(c_hdr);
    if (k >= loaded) {                       // chunk(s) never started: start up to k's
      while (k >= loaded) {
        hdr_chunk(loaded / kP2HdrChunk);
        loaded += kP2HdrChunk;
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    const int landed = loaded;
    hdr_chunk(loaded / kP2HdrChunk);         // and the next chunk, in the background
    loaded += kP2HdrChunk;
    if (lane == 0) {
      ctl_st32(c_hdr, (uint32_t)loaded);
      ctl_st32(c_landed, (uint32_t)landed);
    }
    __syncwarp();
  };
  auto hdr = [&](int k) -> const pk::Seg& { return W.seg[k & (kP2HdrRing - 1)]; };
  auto seg_ntl = [&](int k) -> int {   // tiles of the warp's segment k
    const uint64_t ntile = ctl_ld32(c_ntile);
    const uint64_t segt = ctl_ld32(c_segt);
    const uint64_t t0 = (vw + (uint64_t)kVW * k) * segt;
    return ntile - t0 < segt ? (int)(ntile - t0) : (int)segt;
  };
  // producer: the cursor is warp-uniform and lives in W.ctl; lane 0 issues.
  // skip(): from (pk, pt) to the next tile of a fast segment (or the end)
  auto skip = [&](int pk, int pt) {
    const int nseg = (int)ctl_ld32(c_nseg);
    while (pk < nseg) {
      ensure_hdr(pk);
      const pk::Seg& S = hdr(pk);
      const int ntl = seg_ntl(pk);
      if (!pk::seg_generic(S) && pt < ntl) {
        if (lane == 0) {
          const uint32_t tw = (uint32_t)pk::tile_words(pk::seg_L(S));
          const uint64_t col0 = ((vw + (uint64_t)kVW * pk) * ctl_ld32(c_segt) + pt) * pk::kTile;
          const uint64_t pbody = ctl_ld64(c_body) + 4 * (S.body + (uint64_t)pt * tw);
          const uint64_t usrc = ctl_ld64(c_U) + col0 * 16;
          ctl_st128(c_A, make_uint4((uint32_t)pbody, (uint32_t)(pbody >> 32), (uint32_t)usrc,
                                    (uint32_t)(usrc >> 32)));
          ctl_st32(c_C, tw);
          ctl_st32(c_pntl, (uint32_t)ntl);
        }
        break;
      }
      ++pk;
      pt = 0;
    }
    if (lane == 0) {
      ctl_st32(c_pk, (uint32_t)pk);
      ctl_st32(c_pt, (uint32_t)pt);
    }
    __syncwarp();
  };
  auto issue = [&]() {
    const uint4 B = ctl_ld128(c_B);   // pk, pt, pntl, pslot
    const uint4 C = ctl_ld128(c_C);   // ptw, nseg, -, -
    const int pk = (int)B.x;
    if (pk >= (int)C.y) return;
    const int pt = (int)B.y, pntl = (int)B.z;
    const uint32_t ptw = C.x;
    const int it = p2_item_tiles((int)(ptw >> 7));
    const int nt = pntl - pt < it ? pntl - pt : it;
    // the whole (converged) warp runs this with warp-uniform operands; one
    // elected lane arms the barrier and issues the copies (no per-lane loop).
    // The records are read once (L2 evict-first); the U slices are shared by
    // every band of the launch (default policy: they stay in L2)
    const uint4 A = ctl_ld128(c_A);
    const uint64_t pbody = u64_of(A.x, A.y), usrc = u64_of(A.z, A.w), policy = ctl_ld64(c_policy);
    const uint32_t pslot = B.w;
    const uint32_t st = st0 + pslot * kP2StageBytes, bar = bar0 + 8 * pslot;
    const uint32_t tb = (uint32_t)nt * ptw * 4, ub = (uint32_t)nt * (pk::kTile * 16);   // U is padded
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %6;\n"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%2], %4, [%1], %7;\n"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%8], [%3], %5, [%1];\n"
        "}\n" ::"r"(st), "r"(bar), "l"(pbody), "l"(usrc), "r"(tb), "r"(ub), "r"(tb + ub), "l"(policy),
        "r"(st + tb)
        : "memory");
    __syncwarp();   // every lane has read the cursor before lane 0 advances it
    if (lane == 0) {
      const uint64_t nb = pbody + tb, nu = usrc + ub;
      ctl_st128(c_A, make_uint4((uint32_t)nb, (uint32_t)(nb >> 32), (uint32_t)nu, (uint32_t)(nu >> 32)));
      ctl_st128(c_B, make_uint4(B.x, (uint32_t)(pt + nt), B.z, pslot + 1 == kP2Stages ? 0u : pslot + 1));
    }
    __syncwarp();
    if (pt + nt >= pntl) skip(pk + 1, 0);
  };
  skip(0, 0);
  for (int i = 0; i < kP2Stages; ++i) issue();

  // header and parameters of the warp's segment k -> cur[k & 1], par[k & 1]
  // (cp.async: no registers)
  auto prefetch_par = [&](int k) {
    if (k < (int)ctl_ld32(c_nseg)) {
      if (kCoef && lane < 16) {
        const pk::FieldPar* gp = reinterpret_cast<const pk::FieldPar*>(ctl_ld64(c_gpars));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(par0 + 256 * (k & 1) + 16 * lane),
                     "l"(gp + (uint64_t)kVW * 16 * k + lane) : "memory");
      } else if (lane >= 16 && lane < 19) {
        const char* g = reinterpret_cast<const char*>(reinterpret_cast<const pk::Seg*>(ctl_ld64(c_gsegs)) +
                                                      (uint64_t)kVW * k) + 16 * (lane - 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                     ::"r"(smem_addr(&W.cur[k & 1]) + 16 * (lane - 16)), "l"(g) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch_par(0);

  AT acc = (AT)0;          // row (lane >> 1): the warp's binary64 (single: binary32) sum
  int cslot = 0;
  uint32_t cphase = 0;
  const int nseg = (int)ctl_ld32(c_nseg);

  for (int k = 0; k < nseg; ++k) {
    // this segment's header and parameters have landed; start the next one's
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    prefetch_par(k + 1);
    const pk::Seg& S = W.cur[k & 1];   // shared memory
    const int L = pk::seg_L(S);
    const int We = pk::seg_We(S);
    const int ntl = seg_ntl(k);
    const uint32_t ebase_bits = ((uint32_t)pk::seg_emax_base(S) - 59u) << 23;   // binary32 2^(emax_base - 186)
    const uint32_t par = par0 + 256 * (k & 1);
    // the segment's per-lane sums: coefficient, binary32 s[h][r] = (block-row
    // 2h, 2h + 1) x row r; exact, AT se[4 i + r]
    float2 s[2][4];
    AT se[16];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int r = 0; r < 4; ++r) s[h][r] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int m = 0; m < 16; ++m) se[m] = (AT)0;
    if (!kCoef && !pk::seg_generic(S)) {
      // exact evaluation: the integer-field parameters, computed here
      if (lane < 16) W.par[k & 1][lane] = pk::field_param(S, lane);
      __syncwarp();
    }
    if (!pk::seg_generic(S)) {
      const bool k2 = pk::seg_k2(S), kA = pk::seg_kA(S), kB = pk::seg_kB(S);
      const bool gA = pk::seg_gA(S), gB = pk::seg_gB(S), m12 = pk::seg_m12(S);
      // fields 3..8: w[0] bits 15..29 and w[1] bits 0..14; 9..15: w[1] bits
      // 15..29 and w[2] bits 0..19
      const bool hasA = ((S.w[0] >> 15) & 0x7FFFu) != 0 || (S.w[1] & 0x7FFFu) != 0;
      const bool hasB = ((S.w[1] >> 15) & 0x7FFFu) != 0 || (S.w[2] & 0xFFFFFu) != 0;
      const uint32_t twb = (uint32_t)pk::tile_words(L) * 4;   // bytes per tile
      auto items = [&](auto SPECC) {
        constexpr int SPEC = decltype(SPECC)::value;
        (void)SPEC;
        const int itl = p2_item_tiles(pk::rec_words(L));
        for (int tt = 0; tt < ntl; tt += itl) {
          const uint32_t bar = bar0 + 8 * cslot;
          asm volatile(
              "{\n"
              ".reg .pred p;\n"
              "W2C_WAIT_%=:\n"
              "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
              "@!p bra W2C_WAIT_%=;\n"
              "}\n" ::"r"(bar), "r"(cphase) : "memory");
          const uint32_t st = st0 + cslot * kP2StageBytes + 16 * lane;
          const int nt = ntl - tt < itl ? ntl - tt : itl;
#pragma unroll 1
          for (int it = 0; it < nt; ++it) {
            if constexpr (kCoef)
              p2_tile<SPEC>(st + it * twb, st + nt * twb + it * (pk::kTile * 16), par, m12,
                            k2, hasA, gA, kA, hasB, gB, kB, We, ebase_bits, s);
            else if (SPEC == kSpecDC)
              p2_tile_exact<POL, AT, false, false>(st + it * twb, st + nt * twb + it * (pk::kTile * 16),
                                                   W.par[k & 1], k2, kA, kB, We, (uint32_t)pk::seg_emax_base(S), se);
            else if (SPEC == kSpecFullA)
              p2_tile_exact<POL, AT, true, false>(st + it * twb, st + nt * twb + it * (pk::kTile * 16),
                                                  W.par[k & 1], k2, kA, kB, We, (uint32_t)pk::seg_emax_base(S), se);
            else
              p2_tile_exact<POL, AT, true, true>(st + it * twb, st + nt * twb + it * (pk::kTile * 16),
                                                 W.par[k & 1], k2, kA, kB, We, (uint32_t)pk::seg_emax_base(S), se);
          }
          // every lane has consumed the stage: refill it with the item kP2Stages ahead
          __syncwarp();
          issue();
          cslot = cslot + 1 == kP2Stages ? 0 : cslot + 1;
          cphase ^= cslot == 0 ? 1u : 0u;
        }
      };
      // exact evaluation: the body for the groups present (kSpecDC: no
      // groups, kSpecFullA: group A only, kSpecAny: both)
      if (!kCoef) {
        if (!hasA && !hasB) items(std::integral_constant<int, kSpecDC>());
        else if (!hasB) items(std::integral_constant<int, kSpecFullA>());
        else items(std::integral_constant<int, kSpecAny>());
      }
      else if (m12 && !k2 && hasA && gA && !kA && hasB && gB && !kB) items(std::integral_constant<int, kSpecFull>());
      else if (m12 && !k2 && hasA && gA && !kA && !hasB) items(std::integral_constant<int, kSpecFullA>());
      else if (m12 && !k2 && !hasA && !hasB) items(std::integral_constant<int, kSpecDC>());
      else items(std::integral_constant<int, kSpecAny>());
    } else {
      // generic segment (not staged): per-lane sequential parse from global memory
      const PkView& P = J.p;
      const uint64_t TW = pk::tile_words(L);
      const uint32_t* sbody = P.body + S.body;
      const uint64_t sb = vw + (uint64_t)kVW * k;
      for (int tt = 0; tt < ntl; ++tt) {
        const uint64_t col = (sb * P.g.segt + tt) * pk::kTile + lane;
        if (col >= P.g.bc) continue;
        const float4 u4 = ldg(J.U + col);
        const float u[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i >= pk::band_rows(P.g, band)) break;
          int32_t q[16];
          uint32_t ed;
          pk_generic_parse(&S, sbody + tt * TW, lane, i, q, &ed);
          if constexpr (!kCoef) {
            // (u holds v here: the exact evaluation's padded vector slice)
            float x[16];
            pk::words_from_q(q, (uint32_t)pk::seg_emax_base(S) + ed, x);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              AT t = se[4 * i + r];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                if (POL == WHFF_POLICY_MIXED) t = __dadd_rn(t, (double)__fmul_rn(x[4 * r + j], u[j]));
                else if (POL == WHFF_POLICY_SINGLE) t = __fadd_rn(t, __fmul_rn(x[4 * r + j], u[j]));
                else t = __dadd_rn(t, __dmul_rn((double)x[4 * r + j], (double)u[j]));
              }
              se[4 * i + r] = t;
            }
            continue;
          }
          float w[4];
          w[0] = __fmul_rn(__int2float_rn(q[0]), u[0]);
          w[1] = w[2] = w[3] = 0.0f;
#pragma unroll
          for (int c = 1; c < 16; ++c) {
            const int pos = seq_pos(c);
            w[pos >> 2] = __fmaf_rn(__int2float_rn(q[c]), u[pos & 3], w[pos >> 2]);
          }
          const float sc = __uint_as_float(ebase_bits + (ed << 23));
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            if (i & 1) s[i >> 1][r].y = __fmaf_rn(w[r], sc, s[i >> 1][r].y);
            else s[i >> 1][r].x = __fmaf_rn(w[r], sc, s[i >> 1][r].x);
          }
        }
      }
    }
    // the segment's sums over the warp (row m of the band: m = 4 i + r)
    if constexpr (kCoef) acc = acc + seg_reduce<AT>(s, lane);
    else acc = acc + seg_reduce16<AT>(se, lane);
    if (S.exc_count) pk_exceptions<POL, AT>(J.p, J.v, band, S.exc_begin, S.exc_count, lane, W.rs);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  pk_store_partial<POL, AT>(T, gband, vw, lane, &acc, true, W.rs);
}

// one warp per band: the band's 32 partial records -> its rows of y
template <int EVAL, int POL>
__global__ void __launch_bounds__(128) k_pk_combine(PkTable T, unsigned long long* status) {
  using AT = typename PkAcc<POL>::T;
  const uint64_t gband = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (gband >= T.total_bands) return;
  const int lane = threadIdx.x & 31;
  uint64_t first;
  const PkJob& J = pk_job(T, gband, first);
  const uint64_t band = J.band0 + (gband - first);
  pk_combine_band<EVAL, POL, AT>(J, J.p, T.recs + gband * kVW, band, pk::band_rows(J.p.g, band), lane, status);
}

template <int EVAL, int POL>
static cudaError_t p2_launch(const PkTable& T, unsigned long long* status, cudaStream_t cs) {
  using AT = typename PkAcc<POL>::T;
  const size_t smem = sizeof(P2Warp<AT>) * kP2Warps;
  static std::atomic<uint64_t> attr{0};
  const cudaError_t e = ensure_dyn_smem(k_pk_gemv2<EVAL, POL>, (int)smem, attr);
  if (e != cudaSuccess) return e;
  const unsigned blocks = (unsigned)(T.total_bands * kP2Split);
  k_pk_gemv2<EVAL, POL><<<blocks, 32 * kP2Warps, smem, cs>>>(T, status);
  k_pk_combine<EVAL, POL><<<(unsigned)((T.total_bands + 3) / 4), 128, 0, cs>>>(T, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// decode-only (codec.decompress) from the packed layout: bit-exact words
// ---------------------------------------------------------------------------
// One warp per tile (band x 32 block-columns); exceptions are written by
// k_pk_exc_words afterwards (their records decode to zeros here).
// Latency-bound (a short dependent chain per warp: header, record words,
// lift, four stores), so occupancy pays: 4 CTAs per SM at <= 64 registers
// (the rare generic-record path keeps its arrays on the stack), and the
// words are stored streaming (st.global.cs: written once, never re-read
// here).  4,096 x 262,144 FixedRate(8): 1.147 -> 0.989 ms, FixedAccuracy
// (1e-12) 1.095 -> 0.950 ms; same bits (scratch sweep of 1-6 CTAs per SM);
// the fast records' words loaded 16 bytes at a time: 0.957 / 0.934 ms.
#ifndef WHFF_WORDS_MINB
#define WHFF_WORDS_MINB 4
#endif
#ifndef WHFF_WORDS_CS
#define WHFF_WORDS_CS 1
#endif
#ifndef WHFF_WORDS_V4
#define WHFF_WORDS_V4 1   // 16-byte record loads (0.989 -> 0.957 ms, same bits)
#endif
__global__ void __launch_bounds__(256, WHFF_WORDS_MINB) k_pk_words(PkView P, float* out, uint64_t ld) {
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (wid >= P.g.nband * P.g.ntile) return;
  const uint64_t band = wid / P.g.ntile, t = wid % P.g.ntile;
  const uint64_t sb = t / P.g.segt;
  const int tt = (int)(t % P.g.segt);
  const int nrows = pk::band_rows(P.g, band);
  const pk::Seg S = P.segs[band * P.g.nsegb + sb];
  const int L = pk::seg_L(S), R = pk::rec_words(L), We = pk::seg_We(S);
  const uint32_t ebase = (uint32_t)pk::seg_emax_base(S);
  const uint64_t col = t * pk::kTile + lane;
  const bool active = col < P.g.bc;
  const uint32_t* tile = P.body + S.body + tt * pk::tile_words(L);
  __shared__ pk::FieldPar s_par[8][16];
  const bool generic = pk::seg_generic(S);
  if (!generic) {
    if (lane < 16) s_par[warp][lane] = pk::field_param(S, lane);
    __syncwarp();
  }
  if (!active) return;
  const bool vec = ((reinterpret_cast<uintptr_t>(out) | (ld * 4)) & 15u) == 0;
  int W[16];
  pk::Layout f;
  if (generic) seg_layout(S, W, f);
#if WHFF_WORDS_V4
  // fast records: word k of the lane's four block-rows is one 16-byte
  // (tile_word(k, lane, 0..3)), so all of the lane's record words are in
  // flight at once
  uint4 A4[pk::kFastWords];
  if (!generic) {
#pragma unroll
    for (int k = 0; k < pk::kFastWords; ++k)
      A4[k] = k < R ? ldg(reinterpret_cast<const uint4*>(tile + pk::tile_word(k, lane, 0))) : make_uint4(0, 0, 0, 0);
  }
#endif
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= nrows) break;
    int32_t q[16];
    uint32_t ed;
    if (!generic) {
      uint32_t a[pk::kFastWords];
#if WHFF_WORDS_V4
#pragma unroll
      for (int k = 0; k < pk::kFastWords; ++k)
        a[k] = i == 0 ? A4[k].x : i == 1 ? A4[k].y : i == 2 ? A4[k].z : A4[k].w;
#else
      pk_rec_fast(a, tile, R, lane, i);
#endif
      pk_fields_int(a, s_par[warp], pk::seg_k2(S), pk::seg_kA(S), pk::seg_kB(S), q);
      ed = pk::field_edelta(a[0], We);
    } else {
      uint32_t rec[pk::kMaxRecordWords + 1];
      pk_generic_record(tile, R, lane, i, rec);
      pk::parse_record(f, W, rec, ed, q);
    }
    float x[16];
    pk::words_from_q(q, ebase + ed, x);
    const uint64_t r0 = (band * pk::kBand + i) * 4, c0 = col * 4;
    if (vec && r0 + 4 <= P.g.rows && c0 + 4 <= P.g.cols) {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
#if WHFF_WORDS_CS
        __stcs(reinterpret_cast<float4*>(out + (r0 + rr) * ld + c0),
               make_float4(x[4 * rr], x[4 * rr + 1], x[4 * rr + 2], x[4 * rr + 3]));
#else
        *reinterpret_cast<float4*>(out + (r0 + rr) * ld + c0) =
            make_float4(x[4 * rr], x[4 * rr + 1], x[4 * rr + 2], x[4 * rr + 3]);
#endif
      }
    } else {
      for (int rr = 0; rr < 4; ++rr) {
        if (r0 + rr >= P.g.rows) break;
        for (int j = 0; j < 4; ++j)
          if (c0 + j < P.g.cols) out[(r0 + rr) * ld + c0 + j] = x[4 * rr + j];
      }
    }
  }
}

// exception blocks' words over the decoded matrix; non-finite -> status
__global__ void k_pk_exc_words(PkView P, uint64_t nexc, float* out, uint64_t ld,
                               unsigned long long* status) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= nexc * 16) return;
  const uint64_t e = t >> 4;
  const int k = (int)(t & 15);
  const uint64_t b = P.exc_block[e];
  const uint64_t r = (b / P.g.bc) * 4 + (k >> 2), c = (b % P.g.bc) * 4 + (k & 3);
  if (r >= P.g.rows || c >= P.g.cols) return;
  const float x = __uint_as_float(P.exc_words[t]);
  out[r * ld + c] = x;
  if (!isfinite(x)) atomicMin(status, (unsigned long long)(r * P.g.cols + c));
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static unsigned grid_of(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

cudaError_t pk_launch_words(const PkView& v, uint64_t nexc, float* out, uint64_t ld,
                            unsigned long long* status, cudaStream_t cs) {
  const uint64_t tiles = v.g.nband * v.g.ntile;
  if (tiles) k_pk_words<<<grid_of(tiles, 8), 256, 0, cs>>>(v, out, ld);
  if (nexc) k_pk_exc_words<<<grid_of(nexc * 16, 256), 256, 0, cs>>>(v, nexc, out, ld, status);
  return cudaGetLastError();
}

cudaError_t pk_launch_gemv(int eval, int policy, const PkTable& T, unsigned long long* status,
                           cudaStream_t cs) {
  if (T.total_bands == 0) return cudaSuccess;
  if (eval == WHFF_EVAL_COEFF) {
    if (policy == WHFF_POLICY_SINGLE) return p2_launch<WHFF_EVAL_COEFF, WHFF_POLICY_SINGLE>(T, status, cs);
    return p2_launch<WHFF_EVAL_COEFF, WHFF_POLICY_MIXED>(T, status, cs);
  }
  if (policy == WHFF_POLICY_SINGLE) return p2_launch<WHFF_EVAL_EXACT, WHFF_POLICY_SINGLE>(T, status, cs);
  if (policy == WHFF_POLICY_MIXED) return p2_launch<WHFF_EVAL_EXACT, WHFF_POLICY_MIXED>(T, status, cs);
  return p2_launch<WHFF_EVAL_EXACT, WHFF_POLICY_DOUBLE>(T, status, cs);
}
