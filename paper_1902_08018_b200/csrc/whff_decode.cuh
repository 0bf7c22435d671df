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
#include <type_traits>

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
// count of leading zeros as one FLO.SH (bfind.shiftamt); 0xFFFFFFFF for x == 0
WHFF_HD uint32_t clz_sh(uint32_t x) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("bfind.shiftamt.u32 %0, %1;" : "=r"(d) : "r"(x));
  return d;
#else
  return x ? (uint32_t)__builtin_clz(x) : 0xFFFFFFFFu;
#endif
}
// OR over the lanes currently converged with this one (a superset of the
// lane's own bits, whatever the grouping); the value itself on the host
WHFF_HD uint32_t warp_or(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return __reduce_or_sync(__activemask(), x);
#else
  return x;
#endif
}
// floor(a / d) for 0 <= a < 2^16, 1 <= d <= 16 without the integer-division
// sequence: a * rcp.approx(d) is within 0.02 of a / d, so its truncation is
// the quotient or one less (never more: a non-integer a/d sits >= 1/16 below
// the next integer); one compare fixes it.
WHFF_HD int small_div(int a, int d) {
#if defined(__CUDA_ARCH__)
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)d));
  int q = __float2int_rz(__fmul_rn((float)a, r));
  if ((q + 1) * d <= a) ++q;
  return q;
#else
  return a / d;
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
#if !defined(__CUDA_ARCH__)
inline bool __all_sync(unsigned, bool v) { return v; }   // host check: one lane
#endif

template <typename T>
WHFF_HD T ldg(const T* p) {
#if defined(__CUDA_ARCH__)
  return __ldg(p);
#else
  return *p;
#endif
}

// ---------------------------------------------------------------------------
// 128-bit shift-register bit window over a big-endian (np.packbits,
// MSB-first) bit stream.  w0 holds the next 32 bits; advancing shifts the
// whole register left (four clamped funnel shifts, no compares).  Bits at
// segment positions >= len read as zero: parsing a zero-extended segment
// yields exactly the reference's output (a read past the limit ends the
// block in K:286-368, and zeros never set a magnitude bit, never raise a
// group flag and never form a hit), except for a hit whose sign bit lies past
// the limit, which decode_block handles explicitly (K:353-354).
// ---------------------------------------------------------------------------
WHFF_HD uint32_t fsl(uint32_t hi, uint32_t lo, uint32_t s) {  // s in [0, 32]
#if defined(__CUDA_ARCH__)
  return __funnelshift_lc(lo, hi, s);
#else
  return s >= 32 ? lo : (s ? (hi << s) | (lo >> (32 - s)) : hi);
#endif
}
// low 32 bits of (hi:lo) >> s, s in [0, 32] (clamped)
WHFF_HD uint32_t fsr(uint32_t lo, uint32_t hi, uint32_t s) {
#if defined(__CUDA_ARCH__)
  return __funnelshift_rc(lo, hi, s);
#else
  return s >= 32 ? hi : (s ? (lo >> s) | (hi << (32 - s)) : lo);
#endif
}
// f(std::integral_constant<int, 0..15>) in order, fully unrolled
template <int I = 0, class F>
WHFF_HD void unroll16(F&& f) {
  if constexpr (I < 16) {
    f(std::integral_constant<int, I>());
    unroll16<I + 1>(f);
  }
}
// f(0..15) in order, in groups of four; a group (and everything after it)
// is entered only while `live` has a bit at or above it, so a warp whose
// lanes have no high coefficients skips the rest of the chain in one branch.
template <int G = 0, bool GROUPED = true, class F>
WHFF_HD void unroll16_live(uint32_t live, F&& f) {
  if constexpr (G < 4) {
    f(std::integral_constant<int, 4 * G>());
    f(std::integral_constant<int, 4 * G + 1>());
    f(std::integral_constant<int, 4 * G + 2>());
    f(std::integral_constant<int, 4 * G + 3>());
    if constexpr (G < 3) {
      if (!GROUPED || (live >> (4 * G + 4))) unroll16_live<G + 1, GROUPED>(live, f);
    }
  }
}
WHFF_HD uint32_t top_mask(int nbits) {  // top nbits set (nbits clamped to [0, 32])
#if defined(__CUDA_ARCH__)
  // ~(0xFFFFFFFF >> n) with the funnel shift's clamp at 32: 2 instructions
  return ~__funnelshift_rc(0xFFFFFFFFu, 0u, (uint32_t)max(nbits, 0));
#else
  return nbits <= 0 ? 0u : (nbits >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> nbits));
#endif
}

struct BitWin {
  uint32_t w0, w1, w2, w3;
  int pos;              // segment bits consumed
  int len;              // segment length (bits beyond read as zero)
  int avail;            // REFILL: valid bits held in w0..w3
  const uint32_t* src;  // REFILL: next little-endian payload word
};

// Window at absolute bit `bit` of a payload viewed as LE uint32 words (the
// allocation is padded with >= 32 readable bytes).  The register holds the
// 128 - (bit & 31) bits up to the next word boundary; decode_block<.., false>
// is therefore exact only when (bit & 31) + len <= 128 (see fits_no_refill).
WHFF_HD void win_at(BitWin& b, const uint32_t* words, uint64_t bit, int len) {
  const uint32_t* p = words + (bit >> 5);
  const uint32_t off = (uint32_t)(bit & 31);
  const uint32_t a0 = bswap32(ldg(p)), a1 = bswap32(ldg(p + 1)), a2 = bswap32(ldg(p + 2)),
                 a3 = bswap32(ldg(p + 3));
  b.w0 = fsl(a0, a1, off);
  b.w1 = fsl(a1, a2, off);
  b.w2 = fsl(a2, a3, off);
  b.w3 = fsl(a3, 0u, off);
  b.pos = 0;
  b.len = len;
  b.avail = 128 - (int)off;
  b.src = p + 4;
  if (len < 128) {
    b.w0 &= top_mask(len);
    b.w1 &= top_mask(len - 32);
    b.w2 &= top_mask(len - 64);
    b.w3 &= top_mask(len - 96);
  }
}

// win_at from the four LE payload words already loaded at words + (bit >> 5)
WHFF_HD void win_words(BitWin& b, const uint32_t* words, uint64_t bit, int len, uint32_t x0,
                       uint32_t x1, uint32_t x2, uint32_t x3) {
  const uint32_t off = (uint32_t)(bit & 31);
  const uint32_t a0 = bswap32(x0), a1 = bswap32(x1), a2 = bswap32(x2), a3 = bswap32(x3);
  b.w0 = fsl(a0, a1, off);
  b.w1 = fsl(a1, a2, off);
  b.w2 = fsl(a2, a3, off);
  b.w3 = fsl(a3, 0u, off);
  b.pos = 0;
  b.len = len;
  b.avail = 128 - (int)off;
  b.src = words + (bit >> 5) + 4;
  if (len < 128) {
    b.w0 &= top_mask(len);
    b.w1 &= top_mask(len - 32);
    b.w2 &= top_mask(len - 64);
    b.w3 &= top_mask(len - 96);
  }
}

WHFF_HD bool fits_no_refill(uint64_t bit, int len) { return (int)(bit & 31) + len <= 128; }

// Window from one aligned 16-byte segment (FixedRate(8)).
WHFF_HD void win_128(BitWin& b, uint32_t x, uint32_t y, uint32_t z, uint32_t w, int len) {
  b.w0 = bswap32(x);
  b.w1 = bswap32(y);
  b.w2 = bswap32(z);
  b.w3 = bswap32(w);
  b.pos = 0;
  b.len = len;
  b.avail = 128;
  b.src = nullptr;
  if (len < 128) {
    b.w0 &= top_mask(len);
    b.w1 &= top_mask(len - 32);
    b.w2 &= top_mask(len - 64);
    b.w3 &= top_mask(len - 96);
  }
}

// 128-bit left shift by k < 32 as a chain of 32x32->64 multiply-adds by 2^k:
// (w_i * 2^k + hi(w_{i+1} * 2^k)) runs on the FMA pipe (IMAD.WIDE), leaving
// the ALU pipe -- the decoder's bottleneck -- one shift instead of four.
// x >> J (0 < J < 32, constant) as mul.hi(x, 2^(32-J)): IMAD.HI on the FMA pipe
#ifndef WHFF_SHR_FMA
#define WHFF_SHR_FMA 0
#endif
#ifndef WHFF_ADV_IMAD
#define WHFF_ADV_IMAD 0
#endif
template <int J>
WHFF_HD uint32_t shr_fma(uint32_t x) {
#if defined(__CUDA_ARCH__) && WHFF_SHR_FMA
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "n"(1u << (32 - J)));
  return d;
#else
  return x >> J;
#endif
}
WHFF_HD uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
#if defined(__CUDA_ARCH__)
  uint64_t d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
#else
  return (uint64_t)a * b + c;
#endif
}
WHFF_HD void shl128(BitWin& b, uint32_t k) {
  const uint32_t p = 1u << k;
  const uint64_t t3 = mad_wide(b.w3, p, 0ull);
  const uint64_t t2 = mad_wide(b.w2, p, t3 >> 32);
  const uint64_t t1 = mad_wide(b.w1, p, t2 >> 32);
  const uint64_t t0 = mad_wide(b.w0, p, t1 >> 32);
  b.w3 = (uint32_t)t3;
  b.w2 = (uint32_t)t2;
  b.w1 = (uint32_t)t1;
  b.w0 = (uint32_t)t0;
}

template <bool REFILL>
WHFF_HD void adv(BitWin& b, uint32_t k) {  // k in [0, 32]
  if (WHFF_ADV_IMAD && k < 32) {
    shl128(b, k);
  } else if (!WHFF_ADV_IMAD) {
    b.w0 = fsl(b.w0, b.w1, k);
    b.w1 = fsl(b.w1, b.w2, k);
    b.w2 = fsl(b.w2, b.w3, k);
    b.w3 = fsl(b.w3, 0u, k);
  } else {
    b.w0 = b.w1;
    b.w1 = b.w2;
    b.w2 = b.w3;
    b.w3 = 0u;
  }
  b.pos += (int)k;
  if (REFILL) {
    b.avail -= (int)k;
    if (b.avail < 96) {  // append the next word at register bit `avail`
      const int q = b.pos + b.avail;           // its segment position
      uint32_t wd = bswap32(ldg(b.src));
      b.src++;
      wd &= top_mask(b.len - q);
      const uint32_t sh = (uint32_t)(b.avail - 64);  // 0..31
      b.w2 |= sh ? (wd >> sh) : wd;
      b.w3 = fsl(wd, 0u, 32u - sh);
      b.avail += 32;
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
  t = shr_fma<8>(x); x = (x & ~e.v3) | (t & e.v3);
  t = shr_fma<4>(x); x = (x & ~e.v2) | (t & e.v2);
  t = shr_fma<2>(x); x = (x & ~e.v1) | (t & e.v1);
  t = shr_fma<1>(x); x = (x & ~e.v0) | (t & e.v0);
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

// insert a zero at rank r into both lanes of x (rank r at lane bit 15-r)
WHFF_HD uint32_t insert_zero2(uint32_t x, uint32_t H) {
  uint32_t y = x & ~H;
  return x - y + (y >> 1);
}

// 16 plane words (two 16-bit lanes, see below) -> 16 magnitudes.
// In: X[k] = W_k | W_{k+16} << 16 where W_p bit j = coefficient 15-j of plane p.
// Out: X[j] bit p = plane p bit of coefficient 15-j.
WHFF_HD void transpose16x32(uint32_t X[16]) {
#define WHFF_TSTAGE(J, M)                                            \
  _Pragma("unroll") for (int k = 0; k < 16; ++k) {                   \
    if ((k & (J)) == 0) {                                            \
      uint32_t t = (shr_fma<J>(X[k]) ^ X[k + (J)]) & (M);             \
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

// One plane of the parse (K:323-367); TOP = the plane is the high lane of its
// pair word.  Refinement chunks stay in rank space (bit 31-r / 15-r = rank r).
template <bool REFILL>
struct PlaneParser {
  BitWin& bw;
  uint32_t* pairs;
  uint32_t cur = 0, sig = 0, negm = 0;
  uint32_t nmask = 0, flagbit = 0x80000000u, kq = 1;
  int n = 0;
  bool killed = false;
  WHFF_HD PlaneParser(BitWin& b, uint32_t* p) : bw(b), pairs(p) {}

  template <bool TOP>
  WHFF_HD void plane(int t) {
    const uint32_t x = bw.w0;
    const uint32_t ch = x & nmask;     // refinement chunk (K:326-332)
    cur = TOP ? ch : byte_perm(cur, ch, 0x3276);
    if (!(x & flagbit)) {              // quiet plane: chunk + group flag 0
      adv<REFILL>(bw, kq);
      return;
    }
    adv<REFILL>(bw, (uint32_t)(n + 1));   // significance pass (K:333-367)
    uint32_t rem = ~sig & 0xFFFFu;
    int krem = 16 - n;
    while (true) {
      const uint32_t y = bw.w0;
      const int z = (int)clz32(y);     // insignificant run before the hit
      if (z >= krem) {                 // no hit among the remainder
        adv<REFILL>(bw, (uint32_t)krem);
        break;
      }
      if (bw.pos + z + 1 >= bw.len) {  // sign unavailable: ignore, block ends
        killed = true;
        bw.w0 = bw.w1 = bw.w2 = bw.w3 = 0u;
        bw.len = 0;
        break;
      }
      const uint32_t sgn = (y << (z + 1)) >> 31;
      if (z > 0) rem &= rem - 1;       // skip z insignificant
      if (z > 1) rem &= rem - 1;
      if (z > 2) rem &= rem - 1;
      if (z > 3) {
        rem &= rem - 1;
        for (int i = 4; i < z; ++i) rem &= rem - 1;
      }
      const uint32_t h = rem & (0u - rem);          // the hit
      rem ^= h;                                     // drop the prefix (K:360-363)
      krem -= z + 1;
      const uint32_t r = popc32(sig & (h - 1));    // its rank
      if ((int)r < n) {                             // out of order: shift ranks >= r
        const uint32_t Ht = (0xFFFF0000u << (16 - r)) & 0xFFFF0000u;
        const uint32_t H = Ht | (Ht >> 16);
        cur = insert_zero2(cur, H);
        for (int j = 0; j < (t >> 1); ++j) pairs[j] = insert_zero2(pairs[j], H);
      }
      cur |= (TOP ? 0x80000000u : 0x8000u) >> r;   // significance bit p
      sig |= h;
      if (sgn) negm |= h;
      n += 1;
      if (krem == 0) {                 // remainder empty: no further flag
        adv<REFILL>(bw, (uint32_t)(z + 2));
        break;
      }
      const uint32_t f = (y << (z + 2)) >> 31;     // next group flag
      adv<REFILL>(bw, (uint32_t)(z + 3));
      if (!f) break;
    }
    nmask = top_mask(n);
    flagbit = n < 16 ? (0x80000000u >> n) : 0u;
    kq = (uint32_t)(n + (n < 16));
  }
};

// Parse one block segment (the window's len bits); n_planes is 27 (K:323).
//
// The plane loop is a real loop (small code: the unrolled form overflowed the
// instruction cache).  Refinement chunks are kept in rank space, two planes
// per word: `cur` holds the pair being built, finished pairs go to the
// per-thread array `pairs` (local memory, one store per two planes).  A hit
// whose rank r is below the current count (an out-of-order significance)
// inserts a zero at rank r into every stored pair and into `cur`; in-order
// hits (r == n) need no insertion.  `lanes_mask` is the set of lanes calling
// (for the warp-uniform early exit).
template <bool HAS_RAW, bool REFILL, bool EARLY_EXIT = true>
WHFF_HD void decode_block(BitWin& bw, int planes_limit, Decoded& d, unsigned lanes_mask) {
  const int len = bw.len;
  d.negm = 0;
  d.emax = 0;
  d.raw = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) d.mag[c] = 0;
  bool header_done = true;
  if (len < 9) {                       // K:297-301: header truncated
    d.consumed = len < 0 ? 0 : len;
    header_done = false;
  }
  const uint32_t hdr = bw.w0;
  const uint32_t code = header_done ? hdr >> 23 : 0u;
  d.emax = code;
  if (HAS_RAW && header_done) {
    if (len < 10) {
      d.consumed = 9;
      header_done = false;
    } else {
      adv<REFILL>(bw, 10);
      if ((hdr >> 22) & 1u) {          // K:308-318 raw escape
        d.raw = 1;
        int nw = (len - 10) >> 5;
        if (nw > 16) nw = 16;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          if (c < nw) {
            d.mag[c] = bw.w0;
            adv<REFILL>(bw, 32);
          }
        }
        d.consumed = (len - 10 >= 512) ? 522 : len;
        header_done = false;
      }
    }
  } else if (header_done) {
    adv<REFILL>(bw, 9);
  }
  if (header_done && code == 0) {
    d.consumed = bw.pos;
    header_done = false;
  }
  // lanes without a plane section still walk the (warp-uniform) loop with a
  // zero window so the early-exit vote stays convergent
  if (!header_done) {
    bw.w0 = bw.w1 = bw.w2 = bw.w3 = 0u;
    bw.len = 0;
  }

  uint32_t pairs[14];
  PlaneParser<REFILL> pp(bw, pairs);
  const int pl = planes_limit < kNPlanes ? planes_limit : kNPlanes;
  int t = 0;                           // planes processed (plane P = 26 - t, K:323)
  for (int t2 = 0; t2 < 14; ++t2) {    // two planes per iteration: one word of pairs
    if (t >= pl) break;
    pp.template plane<true>(t);
    if (t + 1 >= pl) {                 // odd plane count: lone top lane
      pairs[t2] = pp.cur;
      t += 1;
      break;
    }
    pp.template plane<false>(t + 1);
    pairs[t2] = pp.cur;
    t += 2;
    if (EARLY_EXIT && __all_sync(lanes_mask, bw.pos >= bw.len)) break;  // all lanes past their data
  }
  const int nstored = (t + 1) >> 1;
  const bool killed = pp.killed;
  const uint32_t sig = pp.sig, negm = pp.negm;
  if (!header_done) return;
  d.consumed = killed ? len : (bw.pos < len ? bw.pos : len);
  d.negm = negm;
  if (sig == 0) return;

  // ranks -> coefficient indices (MSB orientation: bit 31-c = coefficient c)
  const ExpandMasks e = expand_setup(brev32(sig));
  uint32_t C[14];
#pragma unroll
  for (int k = 0; k < 14; ++k) C[k] = k < nstored ? expand2(pairs[k], e) : 0u;
  // X[k] = plane k (low half) | plane k+16 (high half); plane p lives in
  // C[(26-p)>>1], top lane iff (26-p) even; lane bit (15-c) = coefficient c.
  uint32_t X[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int pa = k, pb = k + 16;
    const int ka = (26 - pa) >> 1;
    const bool ta = ((26 - pa) & 1) == 0;
    uint32_t lo = ta ? (C[ka] >> 16) : (C[ka] & 0xFFFFu);
    uint32_t hi = 0;
    if (pb <= 26) {
      const int kb = (26 - pb) >> 1;
      const bool tb = ((26 - pb) & 1) == 0;
      hi = tb ? (C[kb] & 0xFFFF0000u) : (C[kb] << 16);
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


// Signed sequency-order coefficients (|q| < 2^27) -> the 16 lifted integers
// in raster order (codec.py:145-150).
WHFF_HD void lift_signed(const int32_t q[16], int32_t t[16]) {
#pragma unroll
  for (int c = 0; c < 16; ++c) t[seq_pos(c)] = q[c];
#pragma unroll
  for (int i = 0; i < 4; ++i) inv_lift(t[i], t[4 + i], t[8 + i], t[12 + i]);          // columns
#pragma unroll
  for (int i = 0; i < 4; ++i) inv_lift(t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]);  // rows
}

// Lifted integers + emax code -> binary32 words (codec.py:201-206).
WHFF_HD void dequant_words(const int32_t t[16], uint32_t emax, float out[16]) {
  if (emax == 0) {                         // codec.py:205
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = 0.0f;
    return;
  }
  const int k = (int)emax - kEmaxBias - kQuantBits;
  if (dequant_fast_ok(k)) {
    const float s = scale_f32(k);
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = (float)t[i] * s;
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = dequant_slow(t[i], k);
  }
}

// Signed coefficients + emax code -> the 16 binary32 words: the part of
// reconstruct_words after the sign, shared with the packed layout.
WHFF_HD void words_from_signed(const int32_t q[16], uint32_t emax, float out[16]) {
  int32_t t[16];
  lift_signed(q, t);
  dequant_words(t, emax, out);
}

// Decoded block -> 16 binary32 words in raster order (codec.py:209-218).
WHFF_HD void reconstruct_words(const Decoded& d, float out[16]) {
  if (d.raw) {                               // codec.py:215-217
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = as_float(d.mag[i]);
    return;
  }
  int32_t q[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int32_t v = (int32_t)d.mag[c];
    q[c] = ((d.negm >> c) & 1u) ? -v : v;   // codec.py:210-212
  }
  words_from_signed(q, d.emax, out);
}

}  // namespace whff
