// whff_decode.cuh -- WHFZ block decoder (4x4 bit-plane codec) for sm_100a.
//
// Restates, for one block per thread, the reference parse
//   whff/_kernels.pyx:286-368 (_decode_one)     [numpy twin _kernels_py.py:218-287]
// and the reconstruction
//   whff/codec.py:128-134 (_inv_lift), :145-150 (_inverse_transform),
//   :201-206 (_dequantize), :209-218 (_reconstruct_blocks).
//
// Everything here is __host__ __device__ so the exact same code can be
// checked on the CPU against the oracle (tests/test_decoder_host.py) before
// it runs on a B200.
//
// Design: the bitstream is plane-major and its
// significance pass is group-tested, so a thread cannot place refinement bits
// into per-coefficient registers without dynamic register indexing.  Instead:
//   * each plane's refinement chunk is kept in RANK space (bit 31-r = r-th
//     significant coefficient, MSB-first exactly as it sits in the stream),
//     two planes per 32-bit register, in statically indexed registers
//     (the 27-plane loop is unrolled at compile time);
//   * a significance event at rank r inserts a 0 at rank r into every chunk
//     already stored (x - y + (y>>1), y = x & ~H: 3 ops per register) and a 1
//     into the current plane's chunk;
//   * after the parse all chunks live in the final rank space; one SWAR
//     "expand" (PDEP) per register maps ranks to coefficient indices, and a
//     16x32 bit-matrix transpose turns plane masks into 16 magnitudes.
// All costs are fixed per plane / per event, so lanes of a warp (32
// consecutive blocks) stay converged.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define WHFF_HD __host__ __device__ __forceinline__
#else
#define WHFF_HD inline
#endif

namespace whff {

constexpr int kNPlanes = 27;      // codec.py:28
constexpr int kQuantBits = 26;    // codec.py:29
constexpr int kEmaxBias = 160;    // codec.py:30

// codec.py:40  SEQUENCY[i] = raster position of the i-th coefficient
WHFF_HD constexpr int seq_pos(int i) {
  return i == 0 ? 0 : i == 1 ? 1 : i == 2 ? 4 : i == 3 ? 2 : i == 4 ? 5 : i == 5 ? 8
       : i == 6 ? 3 : i == 7 ? 6 : i == 8 ? 9 : i == 9 ? 12 : i == 10 ? 7 : i == 11 ? 10
       : i == 12 ? 13 : i == 13 ? 11 : i == 14 ? 14 : 15;
}

// ---------------------------------------------------------------------------
// portable intrinsics
// ---------------------------------------------------------------------------
WHFF_HD uint32_t clz32(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)__clz((int)x);
#else
  return x ? (uint32_t)__builtin_clz(x) : 32u;
#endif
}
WHFF_HD uint32_t popc32(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)__popc(x);
#else
  return (uint32_t)__builtin_popcount(x);
#endif
}
WHFF_HD uint32_t brev32(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return __brev(x);
#else
  x = ((x >> 1) & 0x55555555u) | ((x & 0x55555555u) << 1);
  x = ((x >> 2) & 0x33333333u) | ((x & 0x33333333u) << 2);
  x = ((x >> 4) & 0x0F0F0F0Fu) | ((x & 0x0F0F0F0Fu) << 4);
  x = ((x >> 8) & 0x00FF00FFu) | ((x & 0x00FF00FFu) << 8);
  return (x >> 16) | (x << 16);
#endif
}
// upper 32 bits of (hi:lo) << s, 0 <= s <= 31
WHFF_HD uint32_t funnel_hi(uint32_t hi, uint32_t lo, uint32_t s) {
#if defined(__CUDA_ARCH__)
  return __funnelshift_l(lo, hi, s);
#else
  return s ? (hi << s) | (lo >> (32 - s)) : hi;
#endif
}
WHFF_HD uint32_t bswap32(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return __byte_perm(x, 0, 0x0123);
#else
  return __builtin_bswap32(x);
#endif
}
// byte permute with the PTX/CUDA selector semantics
WHFF_HD uint32_t byte_perm(uint32_t a, uint32_t b, uint32_t s) {
#if defined(__CUDA_ARCH__)
  return __byte_perm(a, b, s);
#else
  uint64_t v = ((uint64_t)b << 32) | a;
  uint32_t r = 0;
  for (int i = 0; i < 4; ++i) {
    uint32_t sel = (s >> (4 * i)) & 7u;
    r |= (uint32_t)((v >> (8 * sel)) & 0xFFu) << (8 * i);
  }
  return r;
#endif
}
template <typename T>
WHFF_HD T ldg(const T* p) {
#if defined(__CUDA_ARCH__)
  return __ldg(p);
#else
  return *p;
#endif
}

// ---------------------------------------------------------------------------
// Bit window over a big-endian (np.packbits, MSB-first) bit stream.
// w0:w1 always hold the next >= 32 bits starting at bit `off` of w0.
// ---------------------------------------------------------------------------
struct BitWindow {
  uint32_t w0, w1, w2, w3;
  uint32_t off;
  const uint32_t* src;  // next little-endian payload word (REFILL)
};

// Window at absolute bit offset `bit` of a payload viewed as LE uint32 words.
// The payload allocation must be padded with >= 32 readable bytes.
WHFF_HD void window_at(BitWindow& b, const uint32_t* words, uint64_t bit) {
  const uint32_t* p = words + (bit >> 5);
  b.w0 = bswap32(ldg(p));
  b.w1 = bswap32(ldg(p + 1));
  b.w2 = bswap32(ldg(p + 2));
  b.w3 = bswap32(ldg(p + 3));
  b.off = (uint32_t)(bit & 31);
  b.src = p + 4;
}

WHFF_HD uint32_t peek32(const BitWindow& b) { return funnel_hi(b.w0, b.w1, b.off); }

template <bool REFILL>
WHFF_HD void advance(BitWindow& b, uint32_t k) {  // k <= 32
  b.off += k;
  if (b.off >= 32) {
    b.off -= 32;
    b.w0 = b.w1;
    b.w1 = b.w2;
    b.w2 = b.w3;
    if (REFILL) {
      b.w3 = bswap32(ldg(b.src));
      b.src++;
    } else {
      b.w3 = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// SWAR PDEP ("expand", Hacker's Delight 7-5) mirrored to MSB orientation and
// replicated in both 16-bit lanes of a word: deposits the top popc(m) bits of
// each lane into the set positions of the lane mask.
// ---------------------------------------------------------------------------
struct ExpandMasks {
  uint32_t m, v0, v1, v2, v3;
};

WHFF_HD ExpandMasks expand_setup(uint32_t m16_msb) {  // mask in bits 31..16
  ExpandMasks e;
  uint32_t m = m16_msb;
  uint32_t mk = (~m) >> 1;
  uint32_t v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t mp = mk ^ (mk >> 1);
    mp ^= mp >> 2;
    mp ^= mp >> 4;
    mp ^= mp >> 8;
    uint32_t mv = mp & m;
    v[i] = mv;
    m = (m ^ mv) | (mv << (1 << i));
    mk &= ~mp;
  }
  // replicate into the low lane (destinations never cross lanes)
  e.m = m16_msb | (m16_msb >> 16);
  e.v0 = (v[0] & 0xFFFF0000u) | (v[0] >> 16);
  e.v1 = (v[1] & 0xFFFF0000u) | (v[1] >> 16);
  e.v2 = (v[2] & 0xFFFF0000u) | (v[2] >> 16);
  e.v3 = (v[3] & 0xFFFF0000u) | (v[3] >> 16);
  return e;
}

WHFF_HD uint32_t expand2(uint32_t x, const ExpandMasks& e) {
  uint32_t t;
  t = x >> 8; x = (x & ~e.v3) | (t & e.v3);
  t = x >> 4; x = (x & ~e.v2) | (t & e.v2);
  t = x >> 2; x = (x & ~e.v1) | (t & e.v1);
  t = x >> 1; x = (x & ~e.v0) | (t & e.v0);
  return x & e.m;
}

// ---------------------------------------------------------------------------
// Decoded block.  mag[] is in sequency order (codec.py:239); for raw-escape
// blocks mag[] holds the 16 raw IEEE words in raster order (K:303-318).
// ---------------------------------------------------------------------------
struct Decoded {
  uint32_t mag[16];
  uint32_t negm;    // bit c: coefficient c negative
  uint32_t emax;    // 9-bit biased exponent code (0 = zero block)
  uint32_t raw;     // raw escape
  int consumed;     // bits read (K:407)
};

struct ParseState {
  uint32_t C[14];   // rank-space chunks: C[k] top lane = plane 26-2k, low lane = plane 25-2k
  uint32_t sig;     // LSB orientation: bit c = coefficient c significant
  uint32_t negm;
  uint32_t nmask;   // ~(0xFFFFFFFF >> n): the top n bits
  int n;
  int pos;
  bool done;
};

// insert a zero at rank r into both lanes of x (rank r at lane bit 15-r)
WHFF_HD uint32_t insert_zero2(uint32_t x, uint32_t H) {
  uint32_t y = x & ~H;
  return x - y + (y >> 1);
}

template <int P, bool REFILL>
WHFF_HD void plane_step(ParseState& st, BitWindow& bw, int len, int planes_limit) {
  constexpr int K = (26 - P) >> 1;
  constexpr bool TOP = ((26 - P) & 1) == 0;
  if (st.done) return;
  if (st.pos >= len || (26 - P) >= planes_limit) {  // K:323-325
    st.done = true;
    return;
  }
  const int n = st.n;
  const uint32_t x = peek32(bw);
  const int avail = len - st.pos;
  if (avail < n) {  // refinement pass hits the limit (K:328-329)
    uint32_t ch = x & ~(0xFFFFFFFFu >> avail);
    if (TOP) st.C[K] = ch; else st.C[K] |= ch >> 16;
    st.pos = len;
    st.done = true;
    return;
  }
  {
    uint32_t ch = x & st.nmask;   // refinement chunk (K:326-332)
    if (TOP) st.C[K] = ch; else st.C[K] |= ch >> 16;
  }
  if (n >= 16) {
    advance<REFILL>(bw, (uint32_t)n);
    st.pos += n;
    return;
  }
  advance<REFILL>(bw, (uint32_t)n);
  st.pos += n;
  // significance pass (K:333-367)
  uint32_t rem = ~st.sig & 0xFFFFu;
  int krem = 16 - n;
  while (krem > 0) {
    if (st.pos >= len) { st.done = true; return; }
    const uint32_t f = peek32(bw);
    advance<REFILL>(bw, 1);
    st.pos += 1;
    if ((f >> 31) == 0) break;                     // group flag 0: plane ends
    const uint32_t y = f << 1;
    const int z = (int)clz32(y);                   // zero run before the hit
    if (z >= krem) {                               // no hit in the remainder
      if (len - st.pos < krem) { st.pos = len; st.done = true; return; }
      advance<REFILL>(bw, (uint32_t)krem);
      st.pos += krem;
      break;
    }
    if (len - st.pos < z + 1) { st.pos = len; st.done = true; return; }
    advance<REFILL>(bw, (uint32_t)(z + 1));
    st.pos += z + 1;
    if (st.pos >= len) { st.done = true; return; }  // sign unavailable (K:353-354)
    const uint32_t s = (y << (z + 1)) >> 31;
    advance<REFILL>(bw, 1);
    st.pos += 1;
    for (int i = 0; i < z; ++i) rem &= rem - 1;    // skip z insignificant
    const uint32_t h = rem & (0u - rem);           // the hit
    rem ^= h;                                      // drop the prefix (K:360-363)
    krem -= z + 1;
    const uint32_t r = popc32(st.sig & (h - 1));   // its rank
    const uint32_t Ht = (0xFFFF0000u << (16 - r)) & 0xFFFF0000u;  // top r bits of a lane
    const uint32_t H = Ht | (Ht >> 16);
#pragma unroll
    for (int k = 0; k <= K; ++k) st.C[k] = insert_zero2(st.C[k], H);
    st.C[K] |= TOP ? (0x80000000u >> r) : (0x8000u >> r);  // significance bit p
    st.sig |= h;
    if (s) st.negm |= h;
    st.n += 1;
    st.nmask = ~(0xFFFFFFFFu >> st.n);
  }
}

template <int P, bool REFILL>
struct PlaneLoop {
  WHFF_HD static void run(ParseState& st, BitWindow& bw, int len, int pl) {
    plane_step<P, REFILL>(st, bw, len, pl);
    PlaneLoop<P - 1, REFILL>::run(st, bw, len, pl);
  }
};
template <bool REFILL>
struct PlaneLoop<-1, REFILL> {
  WHFF_HD static void run(ParseState&, BitWindow&, int, int) {}
};

// 16 plane words (two 16-bit lanes, see below) -> 16 magnitudes.
// In: X[k] = W_k | W_{k+16} << 16 where W_p bit j = coefficient 15-j of plane p.
// Out: X[j] bit p = plane p bit of coefficient 15-j.
WHFF_HD void transpose16x32(uint32_t X[16]) {
#define WHFF_TSTAGE(J, M)                                            \
  _Pragma("unroll") for (int k = 0; k < 16; ++k) {                   \
    if ((k & (J)) == 0) {                                            \
      uint32_t t = ((X[k] >> (J)) ^ X[k + (J)]) & (M);               \
      X[k] ^= t << (J);                                              \
      X[k + (J)] ^= t;                                               \
    }                                                                \
  }
  WHFF_TSTAGE(8, 0x00FF00FFu)
  WHFF_TSTAGE(4, 0x0F0F0F0Fu)
  WHFF_TSTAGE(2, 0x33333333u)
  WHFF_TSTAGE(1, 0x55555555u)
#undef WHFF_TSTAGE
}

// Parse one block segment of `len` bits.  n_planes is fixed at 27 (K:323).
template <bool HAS_RAW, bool REFILL>
WHFF_HD void decode_block(BitWindow& bw, int len, int planes_limit, Decoded& d) {
  d.negm = 0;
  d.emax = 0;
  d.raw = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) d.mag[c] = 0;
  if (len < 9) {                       // K:297-301: header truncated
    d.consumed = len < 0 ? 0 : len;
    return;
  }
  const uint32_t hdr = peek32(bw);
  const uint32_t code = hdr >> 23;
  advance<REFILL>(bw, 9);
  d.emax = code;
  int pos = 9;
  if (HAS_RAW) {
    if (len < 10) { d.consumed = 9; return; }
    const uint32_t rf = (hdr >> 22) & 1u;
    advance<REFILL>(bw, 1);
    pos = 10;
    if (rf) {                          // K:308-318 raw escape
      d.raw = 1;
      int nw = (len - 10) >> 5;
      if (nw > 16) nw = 16;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        if (c < nw) {
          d.mag[c] = peek32(bw);
          advance<REFILL>(bw, 32);
        }
      }
      d.consumed = (len - 10 >= 512) ? 522 : len;
      return;
    }
  }
  if (code == 0) { d.consumed = pos; return; }

  ParseState st;
#pragma unroll
  for (int k = 0; k < 14; ++k) st.C[k] = 0;
  st.sig = 0;
  st.negm = 0;
  st.nmask = 0;
  st.n = 0;
  st.pos = pos;
  st.done = false;
  PlaneLoop<26, REFILL>::run(st, bw, len, planes_limit);
  d.consumed = st.pos;
  d.negm = st.negm;
  if (st.sig == 0) return;

  // ranks -> coefficient indices (MSB orientation: bit 31-c = coefficient c)
  const ExpandMasks e = expand_setup(brev32(st.sig));
#pragma unroll
  for (int k = 0; k < 14; ++k) st.C[k] = expand2(st.C[k], e);
  // assemble X[k] = plane k (low half) | plane k+16 (high half); a lane value
  // with bit (15-c) = coefficient c is the transpose's column order.
  // plane p lives in C[(26-p)>>1], top lane iff (26-p) even.
  uint32_t X[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int pa = k, pb = k + 16;
    const int ka = (26 - pa) >> 1;
    const bool ta = ((26 - pa) & 1) == 0;
    // low half <- lane of plane pa
    uint32_t lo = ta ? (st.C[ka] >> 16) : (st.C[ka] & 0xFFFFu);
    uint32_t hi = 0;
    if (pb <= 26) {
      const int kb = (26 - pb) >> 1;
      const bool tb = ((26 - pb) & 1) == 0;
      hi = tb ? (st.C[kb] & 0xFFFF0000u) : (st.C[kb] << 16);
    }
    X[k] = lo | hi;
  }
  transpose16x32(X);
#pragma unroll
  for (int j = 0; j < 16; ++j) d.mag[15 - j] = X[j];
}

// ---------------------------------------------------------------------------
// Reconstruction (codec.py:209-218): signed coefficients -> inverse lift
// (columns then rows) -> dequantize -> binary32 words in raster order.
// int32 is exact here: |intermediates| < 2^31 for any 27-plane input
// (tests/test_decoder_host.py::test_lift_range checks the bound).
// ---------------------------------------------------------------------------
WHFF_HD void inv_lift(int32_t& x, int32_t& y, int32_t& z, int32_t& w) {  // codec.py:128-134
  y += w >> 1; w -= y >> 1;
  y += w; w = (int32_t)((uint32_t)w << 1); w -= y;
  z += x; x = (int32_t)((uint32_t)x << 1); x -= z;
  y += z; z = (int32_t)((uint32_t)z << 1); z -= y;
  w += x; x = (int32_t)((uint32_t)x << 1); x -= w;
}

WHFF_HD float as_float(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f;
  __builtin_memcpy(&f, &u, 4);
  return f;
#endif
}
WHFF_HD double as_double(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double f;
  __builtin_memcpy(&f, &u, 8);
  return f;
#endif
}

// binary32(q * 2^k) with a single rounding, as numpy's
// (q.astype(float64) * ldexp(1, k)).astype(float32)  (codec.py:201-206).
// Fast path (k in [-149, 127]): 2^k is a binary32 and fp32(q) is exact
// whenever the product can be subnormal, so one fp32 multiply rounds once.
WHFF_HD bool dequant_fast_ok(int k) { return k >= -149 && k <= 127; }
WHFF_HD float scale_f32(int k) {
  return as_float(k >= -126 ? (uint32_t)(k + 127) << 23 : 1u << (k + 149));
}
WHFF_HD float dequant_slow(int32_t q, int k) {
  // exact 2^k in binary64 (k in [-186, 325] here)
  return (float)((double)q * as_double((uint64_t)(k + 1023) << 52));
}


// Decoded block -> 16 binary32 words in raster order (codec.py:209-218).
WHFF_HD void reconstruct_words(const Decoded& d, float out[16]) {
  if (d.raw) {                               // codec.py:215-217
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = as_float(d.mag[i]);
    return;
  }
  int32_t t[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int32_t v = (int32_t)d.mag[c];
    t[seq_pos(c)] = ((d.negm >> c) & 1u) ? -v : v;   // codec.py:210-212
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) inv_lift(t[i], t[4 + i], t[8 + i], t[12 + i]);          // columns
#pragma unroll
  for (int i = 0; i < 4; ++i) inv_lift(t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]);  // rows
  if (d.emax == 0) {                         // codec.py:205
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = 0.0f;
    return;
  }
  const int k = (int)d.emax - kEmaxBias - kQuantBits;
  if (dequant_fast_ok(k)) {
    const float s = scale_f32(k);
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = (float)t[i] * s;
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = dequant_slow(t[i], k);
  }
}

}  // namespace whff
