// whff_packed.cuh -- the tile-packed device layout of a WHFZ stream and the
// fused decode + GEMV / decode-only kernels that read it.
//
// Why a second device layout.  The reference bitstream (codec.py:225-314,
// K:139-368) codes every 4x4 block as bit planes with group-tested
// significance: each block is a serial parse whose cost is ~1,000 thread
// instructions per 16-byte block on a B200, 11x the ~90 the
// SM can issue per block at HBM speed.  The information the GEMV needs per
// block is only (emax, 16 signed integer coefficients q_c) -- exactly what
// the reference's decode_blocks (K:371-408) hands to _reconstruct_blocks
// (codec.py:209-218).  At upload time this layout re-codes those values
// losslessly so that decoding is branch-free SIMT work:
//
//   band     = 4 block-rows (16 matrix rows)
//   tile     = band x 32 block-columns; lane l of a warp owns block-column
//              32 t + l of every block-row of the band
//   segment  = band x up to 8 or 16 tiles (per stream) sharing one "field
//              profile": a width W_c per coefficient c (sequency order,
//              codec.py:40) = the widest value of c in the segment, and a
//              width W_e for emax - emax_base
//   record   = one block: [emax delta: W_e bits][field 0 .. field 15], the
//              fields at offsets fixed per segment; field 0 (DC) is two's
//              complement, fields 1..15 offset-binary (q + 2^(W-1)).
//
// Records are MSB-first bit strings of L bits (L per segment), stored in
// R = ceil(L / 32) whole 32-bit words.  A tile holds the records of its 4
// block-rows x 32 block-columns word-major: word k of the record of (row i,
// lane l) is tile word (32 k + l) * 4 + i, so one 16-byte shared-memory
// load by lane l yields word k of all four rows (rows past the band's end
// are zero records).  A tile is 128 R words; a segment body is its tiles.
//
// Fast path (every segment of a smooth WHFF operator, L <= 160): field c is
// read from a register pair (a_k, a_k+1) of the record's five words chosen
// per segment from two candidates: k = 0 for c <= 1, 0 or 1 for c = 2
// (flag k2), 1 or 2 for c = 3..8 (flag kA), 2 or 3 for c = 9..15 (flag kB)
// (the packer pads so each field lies inside its pair), with two funnel
// shifts: the left one brings the field to the top, the right one shifts it
// down under the binary32 exponent of 2^23 ("magic number"), so
// float(2^23 + u) - (2^23 + 2^(W-1)) = q exactly (W <= 23).  Segments whose
// fields do not fit (adversarial data) take a generic per-lane path.
//
// Blocks the coefficient-domain evaluation cannot take (raw escapes, scales
// outside 2^-126..2^100; see coef_ok in whff_b200.cu) are "exceptions":
// their records are zero and their 16 decoded binary32 words (bit-exact
// with codec.decompress) live in a side list processed per segment.
//
// Everything the packer and the kernels share is __host__ __device__.
#pragma once

#include <cmath>
#include <cstring>

#include "whff_decode.cuh"

namespace whff {
namespace pk {

constexpr int kBand = 4;          // block-rows per band
constexpr int kTile = 32;         // block-columns per tile (one per lane)
// Tiles per segment, chosen per stream at pack time (seg_tiles_for_mode):
// 16 for the variable-rate modes (short records: per-segment control is a
// large share, and the field widths barely grow), 8 for FixedRate (longer
// segments widen its fields enough to cost more than they save).
constexpr int kSegTilesRate = 8;
constexpr int kSegTilesVar = 16;
constexpr int kSegTiles = kSegTilesVar;   // the largest (tests/fused_order.py seg_tiles_for)
WHFF_HD int seg_tiles_for_mode(int mode) { return mode == 0 ? kSegTilesRate : kSegTilesVar; }
constexpr int kMagicW = 23;       // widest offset-binary field on the magic path
constexpr int kMaxRecordBits = 9 + 28 * 16;
constexpr int kMaxRecordWords = (kMaxRecordBits + 31) / 32;   // 15
constexpr int kFastWords = 5;                                 // fast path: L <= 160
constexpr uint32_t kMagic = 0x4B000000u;                      // binary32 2^23

// Segment header (48 bytes).
struct alignas(16) Seg {
  uint64_t body;       // word offset of the segment body
  uint32_t hdr;        // [0:9) emax_base [9:13) W_e [13] generic [14] k2 [15] kA [16:25) L [25] kB
                       // [26] gA [27] gB (group path: the group spans <= 23 bits)
                       // [28] m12 (c = 1, 2 no wider than the magic path: k_pk_gemv2
                       //      converts them like c >= 3)
  uint32_t w[3];       // W_c, 5 bits each: c = 6 * word + slot
  uint32_t o[4];       // fast path: offset of field c (8 bits): c = 4 * word + slot
  uint32_t exc_begin;  // first exception of the segment
  uint32_t exc_count;
};

WHFF_HD int seg_emax_base(const Seg& s) { return (int)(s.hdr & 511u); }
WHFF_HD int seg_We(const Seg& s) { return (int)((s.hdr >> 9) & 15u); }
WHFF_HD bool seg_generic(const Seg& s) { return (s.hdr >> 13) & 1u; }
WHFF_HD bool seg_k2(const Seg& s) { return (s.hdr >> 14) & 1u; }
WHFF_HD bool seg_kA(const Seg& s) { return (s.hdr >> 15) & 1u; }
WHFF_HD bool seg_kB(const Seg& s) { return (s.hdr >> 25) & 1u; }
WHFF_HD bool seg_gA(const Seg& s) { return (s.hdr >> 26) & 1u; }
WHFF_HD bool seg_gB(const Seg& s) { return (s.hdr >> 27) & 1u; }
WHFF_HD bool seg_m12(const Seg& s) { return (s.hdr >> 28) & 1u; }
WHFF_HD int seg_L(const Seg& s) { return (int)((s.hdr >> 16) & 511u); }
WHFF_HD int seg_W(const Seg& s, int c) { return (int)((s.w[c / 6] >> (5 * (c % 6))) & 31u); }
WHFF_HD int seg_o(const Seg& s, int c) { return (int)((s.o[c / 4] >> (8 * (c % 4))) & 255u); }

// register pair of field c on the fast path (the segment's flags)
WHFF_HD int field_pair(int c, bool k2, bool kA, bool kB) {
  return c <= 1 ? 0 : c == 2 ? (k2 ? 1 : 0) : c <= 8 ? (kA ? 2 : 1) : (kB ? 3 : 2);
}

// Field offsets from the widths (W[0] >= 1).  Fast layout: fields in order,
// each inside the 64-bit window of its register pair (bits [32k, 32k + 64)
// of the record; padded up to 32k when needed), a group (c = 2, 3..8,
// 9..15) taking its second candidate pair only when the first cannot hold
// it; generic (fields back to back) when a field does not fit, a field
// c >= 3 is wider than the magic path allows, or L > 160.
struct Layout {
  int We, L;
  bool fast, k2, kA, kB, gA, gB, m12;
  int o[16];
};
WHFF_HD bool place_group(const int W[16], int c0, int c1, int k, int& cur, int o[16]) {
  int any = 0;
  for (int c = c0; c <= c1; ++c) any |= W[c];
  if (!any) {   // an absent group takes no bits (and does not move the cursor)
    for (int c = c0; c <= c1; ++c) o[c] = 0;
    return true;
  }
  int x = cur < 32 * k ? 32 * k : cur;
  for (int c = c0; c <= c1; ++c) {
    if (W[c] == 0) { o[c] = 0; continue; }
    if (x + W[c] > 32 * k + 64) return false;
    o[c] = x;
    x += W[c];
  }
  cur = x;
  return true;
}
WHFF_HD void make_layout(int We, const int W[16], Layout& f) {
  int cur = We;
  bool fast = true;
  f.k2 = f.kA = f.kB = false;
  for (int c = 0; c < 16; ++c) f.o[c] = 0;
  for (int c = 3; c < 16; ++c)
    if (W[c] > kMagicW) fast = false;   // (c = 1, 2 convert as integers)
  if (fast) fast = place_group(W, 0, 1, 0, cur, f.o);
  if (fast) {
    int t = cur, o2[16];
    if (place_group(W, 2, 2, 0, t, o2)) { f.o[2] = o2[2]; cur = t; }
    else { f.k2 = true; fast = place_group(W, 2, 2, 1, cur, f.o); }
  }
  if (fast) {
    int t = cur, oA[16];
    if (place_group(W, 3, 8, 1, t, oA)) { for (int c = 3; c <= 8; ++c) f.o[c] = oA[c]; cur = t; }
    else { f.kA = true; fast = place_group(W, 3, 8, 2, cur, f.o); }
  }
  if (fast) {
    int t = cur, oB[16];
    if (place_group(W, 9, 15, 2, t, oB)) { for (int c = 9; c <= 15; ++c) f.o[c] = oB[c]; cur = t; }
    else { f.kB = true; fast = place_group(W, 9, 15, 3, cur, f.o); }
  }
  if (!fast) {
    f.k2 = f.kA = f.kB = false;
    cur = We;
    for (int c = 0; c < 16; ++c) {
      f.o[c] = cur;
      cur += W[c];
    }
  }
  f.We = We;
  f.L = cur;
  f.fast = fast;
  int wa = 0, wb = 0;
  for (int c = 3; c <= 8; ++c) wa += W[c];
  for (int c = 9; c < 16; ++c) wb += W[c];
  f.gA = fast && wa <= kMagicW;
  f.gB = fast && wb <= kMagicW;
  f.m12 = fast && W[1] <= kMagicW && W[2] <= kMagicW;
}

// segment header word from a layout
WHFF_HD uint32_t seg_hdr(uint32_t ebase, const Layout& f) {
  return ebase | ((uint32_t)f.We << 9) | ((f.fast ? 0u : 1u) << 13) | ((f.k2 ? 1u : 0u) << 14) |
         ((f.kA ? 1u : 0u) << 15) | ((uint32_t)f.L << 16) | ((f.kB ? 1u : 0u) << 25) |
         ((f.gA ? 1u : 0u) << 26) | ((f.gB ? 1u : 0u) << 27) | ((f.m12 ? 1u : 0u) << 28);
}

// signed width: the fewest bits holding q in two's complement / offset binary
WHFF_HD int qwidth(int32_t q) {
  if (q == 0) return 0;
  const uint32_t a = (uint32_t)(q >= 0 ? q : ~q);
  return a == 0 ? 1 : 33 - (int)clz32(a);
}
WHFF_HD int bitwidth_u(uint32_t x) { return x == 0 ? 0 : 32 - (int)clz32(x); }

// words of one record / tile (4 row slots x 32 lanes)
WHFF_HD int rec_words(int L) { return (L + 31) >> 5; }
WHFF_HD uint64_t tile_words(int L) { return 128ull * (uint64_t)rec_words(L); }
// tile word holding word k of the record of (row i, lane l)
WHFF_HD uint32_t tile_word(int k, int lane, int i) { return ((uint32_t)(32 * k + lane) << 2) | (uint32_t)i; }

// Geometry of a packed stream.
struct Geom {
  uint64_t rows, cols, br, bc;
  uint64_t nband;   // ceil(br / 4)
  uint64_t ntile;   // tiles per band: ceil(bc / 32)
  uint64_t nsegb;   // segments per band: ceil(ntile / segt)
  uint64_t segt;    // tiles per segment
};
WHFF_HD Geom make_geom(uint64_t rows, uint64_t cols, int segt) {
  Geom g;
  g.segt = (uint64_t)segt;
  g.rows = rows;
  g.cols = cols;
  g.br = (rows + 3) / 4;
  g.bc = (cols + 3) / 4;
  g.nband = (g.br + kBand - 1) / kBand;
  g.ntile = (g.bc + kTile - 1) / kTile;
  g.nsegb = (g.ntile + g.segt - 1) / g.segt;
  return g;
}
WHFF_HD int band_rows(const Geom& g, uint64_t band) {
  const uint64_t r = g.br - band * kBand;
  return r < (uint64_t)kBand ? (int)r : kBand;
}
WHFF_HD int seg_tiles(const Geom& g, uint64_t sb) {
  const uint64_t r = g.ntile - sb * g.segt;
  return r < g.segt ? (int)r : (int)g.segt;
}

// record bits: put the low W bits of val at record bits [pos, pos + W)
WHFF_HD void put_bits(uint32_t* rec, int pos, int W, uint32_t val) {
  if (W <= 0) return;
  const uint64_t v = (uint64_t)(val & (W >= 32 ? 0xFFFFFFFFu : ((1u << W) - 1u))) << (64 - W);
  const int w = pos >> 5, s = pos & 31;
  const uint64_t sh = v >> s;
  rec[w] |= (uint32_t)(sh >> 32);
  if (s + W > 32) rec[w + 1] |= (uint32_t)sh;
}
// W bits at record bits [pos, pos + W), W <= 32, unsigned
WHFF_HD uint32_t get_bits(const uint32_t* rec, int pos, int W) {
  if (W <= 0) return 0u;
  const int w = pos >> 5, s = pos & 31;
  const uint32_t hi = rec[w], lo = (s + W > 32) ? rec[w + 1] : 0u;
  const uint32_t x = fsl(hi, lo, (uint32_t)s);
  return W >= 32 ? x : x >> (32 - W);
}

// Record of one decoded block (q in sequency order) under a layout.
WHFF_HD void build_record(const Layout& f, const int W[16], uint32_t edelta, const int32_t q[16],
                          uint32_t* rec /* kMaxRecordWords, zeroed */) {
  put_bits(rec, 0, f.We, edelta);
  for (int c = 0; c < 16; ++c) {
    if (W[c] == 0) continue;
    const uint32_t u = c == 0 ? (uint32_t)q[c] : (uint32_t)(q[c] + (1 << (W[c] - 1)));
    put_bits(rec, f.o[c], W[c], u);
  }
}
// ...and its inverse (both paths: offsets from the layout)
WHFF_HD void parse_record(const Layout& f, const int W[16], const uint32_t* rec, uint32_t& edelta,
                          int32_t q[16]) {
  edelta = get_bits(rec, 0, f.We);
  for (int c = 0; c < 16; ++c) {
    if (W[c] == 0) {
      q[c] = 0;
      continue;
    }
    const uint32_t u = get_bits(rec, f.o[c], W[c]);
    if (c == 0) q[c] = (int32_t)(u << (32 - W[c])) >> (32 - W[c]);
    else q[c] = (int32_t)u - (1 << (W[c] - 1));
  }
}

// Coefficient-domain exceptions (codec.py:215-217 raw escapes; scales the
// binary32 sink cannot hold): identical to coef_ok() in whff_b200.cu.
WHFF_HD bool is_exception(const Decoded& d) {
  const int k = (int)d.emax - kEmaxBias - kQuantBits;
  return d.raw || (d.emax != 0 && !(k >= -126 && k <= 100));
}

WHFF_HD void signed_coefs(const Decoded& d, int32_t q[16]) {
  for (int c = 0; c < 16; ++c) {
    const int32_t m = (int32_t)d.mag[c];
    q[c] = ((d.negm >> c) & 1u) ? -m : m;
  }
}

// Words of a block from its signed coefficients (as reconstruct_words).
WHFF_HD void words_from_q(const int32_t q[16], uint32_t emax, float out[16]) {
  words_from_signed(q, emax, out);
}

// ---------------------------------------------------------------------------
// fast-path field extraction (shared by the kernels and the host check)
// ---------------------------------------------------------------------------
// Per-field parameters (a warp keeps them in shared memory):
// c = 0 (DC, two's complement): {W_e (left shift), 32 - W_0 (arithmetic
// right shift), -, -}.  c = 1, 2 (the large AC coefficients, up to 28 bits,
// converted as integers): {left shift inside the static pair (0..63), 0,
// 32 - W, 2^(W-1)}.  c >= 3 (W <= 23): {left shift, 2^23 >> W (high word of
// the magic right funnel), 32 - W (its shift), bits of -(2^23 + 2^(W-1))}.
// Absent fields give q = 0 on both paths.
struct alignas(16) FieldPar {
  uint32_t x, y, z, w;
};
WHFF_HD FieldPar field_param(const Seg& S, int c) {
  const int W = seg_W(S, c);
  FieldPar p;
  if (c == 0) {
    p.x = (uint32_t)seg_We(S);
    p.y = 32u - (uint32_t)W;
    p.z = 0u;
    p.w = 0u;
  } else if (W == 0) {
    p.x = 0u;
    p.y = c <= 2 ? 0u : kMagic;
    p.z = 32u;
    p.w = c <= 2 ? 0u : 0xCB000000u;         // -2^23
  } else {
    const int k = field_pair(c, seg_k2(S), seg_kA(S), seg_kB(S));
    p.x = (uint32_t)(seg_o(S, c) - 32 * k);
    p.y = c <= 2 ? 0u : kMagic >> W;
    p.z = 32u - (uint32_t)W;
    p.w = c <= 2 ? 1u << (W - 1) : 0xCB000000u + (1u << (W - 1));   // -(2^23 + 2^(W-1))
  }
  return p;
}

// Group extraction (c = 3..8 "A", 9..15 "B"), used when a group's fields
// span at most 23 bits together: one 64-bit right shift brings the whole
// group to the bottom of a register (x = (hi:lo) >> n), then each field is
// one LOP3 -- (x & mask) | 2^23-exponent -- giving the binary32 value
// 2^23 + u 2^s exactly, and q = value 2^-s - (2^(23-s) + 2^(W-1)) exactly
// (one FMA: every intermediate is an exact binary32 integer).  Parameters:
// {mask = (2^W - 1) << s, bits of 2^-s, bits of -(2^(23-s) + 2^(W-1)), n};
// absent fields {0, 1.0, -2^23, n} give q = 0.
WHFF_HD constexpr int group_first(int g) { return g == 0 ? 3 : 9; }
WHFF_HD constexpr int group_last(int g) { return g == 0 ? 8 : 15; }
WHFF_HD uint32_t f32_bits(float x) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(x);
#else
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return u;
#endif
}
WHFF_HD int group_width(const Seg& S, int g) {
  int w = 0;
  for (int c = group_first(g); c <= group_last(g); ++c) w += seg_W(S, c);
  return w;
}
WHFF_HD bool group_magic(const Seg& S, int g) { return g == 0 ? seg_gA(S) : seg_gB(S); }
WHFF_HD FieldPar group_param(const Seg& S, int c) {
  const int g = c <= 8 ? 0 : 1;
  const int k = field_pair(c, seg_k2(S), seg_kA(S), seg_kB(S));
  int end = 0;   // end bit (exclusive) of the group inside the pair window
  for (int cc = group_first(g); cc <= group_last(g); ++cc) {
    const int Wc = seg_W(S, cc);
    if (Wc && seg_o(S, cc) - 32 * k + Wc > end) end = seg_o(S, cc) - 32 * k + Wc;
  }
  FieldPar p;
  p.w = end ? (uint32_t)(64 - end) : 0u;
  const int W = seg_W(S, c);
  const int sh = W ? end - (seg_o(S, c) - 32 * k + W) : 0;
  p.x = W ? ((W >= 32 ? 0xFFFFFFFFu : ((1u << W) - 1u)) << sh) : 0u;
  p.y = (uint32_t)(127 - sh) << 23;                            // 2^-sh
  p.z = W ? 0x80000000u | f32_bits((float)((1u << (23 - sh)) + (1u << (W - 1)))) : 0xCB000000u;
  return p;
}
// the parameters k_pk_gemv2 uses for field c of a fast segment (the packer
// stores them per segment: whff_dstream_pack)
WHFF_HD FieldPar seg_param(const Seg& S, int c) {
  if (c >= 3 && group_magic(S, c <= 8 ? 0 : 1)) return group_param(S, c);
  if ((c == 1 || c == 2) && seg_m12(S)) {
    // the magic-number format of c >= 3 (W <= 23: the binary32 value is exact)
    const int W = seg_W(S, c);
    FieldPar p;
    if (W == 0) {
      p.x = 0u;
      p.y = kMagic;
      p.z = 32u;
      p.w = 0xCB000000u;
    } else {
      const int k = field_pair(c, seg_k2(S), seg_kA(S), seg_kB(S));
      p.x = (uint32_t)(seg_o(S, c) - 32 * k);
      p.y = kMagic >> W;
      p.z = 32u - (uint32_t)W;
      p.w = 0xCB000000u + (1u << (W - 1));
    }
    return p;
  }
  return field_param(S, c);
}

// the group bits at the bottom of a register
WHFF_HD uint32_t group_bits(uint32_t hi, uint32_t lo, uint32_t n) {
  return (uint32_t)((((uint64_t)hi << 32) | lo) >> n);
}
WHFF_HD float group_field_f(uint32_t x, const FieldPar& p) {
  const uint32_t b = (x & p.x) | kMagic;
#if defined(__CUDA_ARCH__)
  return __fmaf_rn(__uint_as_float(b), __uint_as_float(p.y), __uint_as_float(p.z));
#else
  return std::fma(as_float(b), as_float(p.y), as_float(p.z));
#endif
}

// high word of the 64-bit (hi:lo) << n, n in [0, 63]: one SHF.L.U64.HI
WHFF_HD uint32_t fsl64(uint32_t hi, uint32_t lo, uint32_t n) {
  return (uint32_t)(((((uint64_t)hi << 32) | lo) << n) >> 32);
}

// Field c >= 1 read from its register pair (hi, lo): the 64-bit left shift
// brings it to the top, the clamped right funnel shifts it under the
// exponent of 2^23, so the binary32 bits are 2^23 + u exactly; minus
// 2^23 + 2^(W-1) = q.
WHFF_HD float field_f(uint32_t hi, uint32_t lo, const FieldPar& p) {
  const uint32_t x = fsl64(hi, lo, p.x);
  const uint32_t fb = fsr(x, p.y, p.z);
#if defined(__CUDA_ARCH__)
  return __fadd_rn(__uint_as_float(fb), __uint_as_float(p.w));
#else
  return as_float(fb) + as_float(p.w);
#endif
}
WHFF_HD int32_t field_i(uint32_t hi, uint32_t lo, const FieldPar& p) {
  const uint32_t fb = fsr(fsl64(hi, lo, p.x), p.y, p.z);
  return (int32_t)(fb - (p.w & 0x7FFFFFFFu));
}
WHFF_HD int32_t field_dc(uint32_t a0, uint32_t a1, const FieldPar& p0) {
  return (int32_t)fsl64(a0, a1, p0.x) >> p0.y;
}
WHFF_HD uint32_t field_edelta(uint32_t a0, int We) { return fsr(a0, 0u, 32u - (uint32_t)We); }

// All 16 coefficients (sequency order) of one fast-path record a[0..3]
// (the host check's form; the kernels read par from shared memory).
WHFF_HD void fields_int(const uint32_t a[kFastWords], const FieldPar par[16], bool k2, bool kA, bool kB,
                        int32_t q[16]) {
  q[0] = field_dc(a[0], a[1], par[0]);
  for (int c = 1; c < 16; ++c) {
    const int k = field_pair(c, k2, kA, kB);
    q[c] = field_i(a[k], k + 1 < kFastWords ? a[k + 1] : 0u, par[c]);
  }
}
}  // namespace pk
}  // namespace whff
static_assert(sizeof(whff::pk::Seg) == 48, "segment header is 48 bytes");
