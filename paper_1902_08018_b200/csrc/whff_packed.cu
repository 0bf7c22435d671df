// whff_packed.cu -- kernels of the tile-packed layout (whff_packed.cuh):
// the packer (reference / skeleton-first stream -> packed), the fused
// decode + GEMV that reads it (the hot path), decode-only words, and the
// exception side list, and their host launchers (whff_packed_api.h).
#include <cstdlib>
#include <type_traits>

#include "whff_common.cuh"
#include "whff_packed.cuh"
#include "whff_packed_api.h"

// field widths / layout of a segment header
__device__ __forceinline__ void seg_layout(const pk::Seg& S, int W[16], pk::Layout& f) {
#pragma unroll
  for (int c = 0; c < 16; ++c) W[c] = pk::seg_W(S, c);
  pk::make_layout(pk::seg_We(S), W, f);
}

// Record words a[i][0..3] of the lane's block in each of the 4 band rows of a
// tile: mf full words (interleaved) and the packed tail; absent words 0.
// (Rows past the band's end read neighbouring data: discarded.)
__device__ __forceinline__ uint32_t pk_tail(const uint32_t* rb, int mf, int tb, uint32_t toff, uint32_t tsh) {
  if (!tb) return 0u;
  const uint32_t* p = rb + 32 * mf + toff;
  return fsl(ldg(p), ldg(p + 1), tsh);
}
__device__ __forceinline__ void pk_load4(uint32_t a[4][4], const uint32_t* base, int L, int mf, int tb,
                                         uint32_t toff, uint32_t tsh, int lane) {
  switch (mf) {
    case 0:
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t* rb = base + i * L;
        a[i][0] = pk_tail(rb, 0, tb, toff, tsh);
        a[i][1] = a[i][2] = a[i][3] = 0u;
      }
      break;
    case 1:
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t* rb = base + i * L;
        a[i][0] = ldg(rb + lane);
        a[i][1] = pk_tail(rb, 1, tb, toff, tsh);
        a[i][2] = a[i][3] = 0u;
      }
      break;
    case 2:
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t* rb = base + i * L;
        a[i][0] = ldg(rb + lane);
        a[i][1] = ldg(rb + 32 + lane);
        a[i][2] = pk_tail(rb, 2, tb, toff, tsh);
        a[i][3] = 0u;
      }
      break;
    case 3:
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t* rb = base + i * L;
        a[i][0] = ldg(rb + lane);
        a[i][1] = ldg(rb + 32 + lane);
        a[i][2] = ldg(rb + 64 + lane);
        a[i][3] = pk_tail(rb, 3, tb, toff, tsh);
      }
      break;
    default:
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t* rb = base + i * L;
        a[i][0] = ldg(rb + lane);
        a[i][1] = ldg(rb + 32 + lane);
        a[i][2] = ldg(rb + 64 + lane);
        a[i][3] = ldg(rb + 96 + lane);
      }
      break;
  }
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

// All 16 coefficients (sequency order) of one fast-path record.
__device__ __forceinline__ void pk_fields_int(const uint32_t a[4], const pk::FieldPar* par /* smem */, bool k2,
                                              int32_t q[16]) {
  q[0] = pk::field_dc(a[0], a[1], lds_par(par));
  q[1] = pk::field_i(a[0], a[1], lds_par(par + 1));
  q[2] = k2 ? pk::field_i(a[1], a[2], lds_par(par + 2)) : pk::field_i(a[0], a[1], lds_par(par + 2));
#pragma unroll
  for (int c = 3; c <= 8; ++c) q[c] = pk::field_i(a[1], a[2], lds_par(par + c));
#pragma unroll
  for (int c = 9; c < 16; ++c) q[c] = pk::field_i(a[2], a[3], lds_par(par + c));
}

// Generic path: the lane's whole record (any L) into rec[], then parse.
__device__ __noinline__ void pk_generic_record(const uint32_t* rb, int L, int lane, uint32_t* rec) {
  const int mf = L >> 5, tb = L & 31;
  for (int k = 0; k <= pk::kMaxRecordWords; ++k) rec[k] = 0u;
  for (int k = 0; k < mf; ++k) rec[k] = ldg(rb + 32 * k + lane);
  if (tb) {
    const uint32_t bit = (uint32_t)lane * tb;
    const uint32_t* p = rb + 32 * mf + (bit >> 5);
    rec[mf] = fsl(ldg(p), ldg(p + 1), bit & 31) & ~(0xFFFFFFFFu >> tb);
  }
}

// ---------------------------------------------------------------------------
// fused decode + GEMV over packed streams (the hot path)
// ---------------------------------------------------------------------------
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


// Generic segments (fields wider than the fast path allows, L up to 457):
// one record parsed sequentially; out of line, results through memory.
__device__ __noinline__ void pk_generic_parse(const pk::Seg* Sp, const uint32_t* rb, int lane, int32_t* q,
                                              uint32_t* ed) {
  const pk::Seg S = *Sp;
  int W[16];
  pk::Layout f;
  seg_layout(S, W, f);
  uint32_t rec[pk::kMaxRecordWords + 1];
  pk_generic_record(rb, f.L, lane, rec);
  pk::parse_record(f, W, rec, *ed, q);
}

// one fast-path record (the exact evaluation re-reads it per row from L1)
__device__ __forceinline__ void pk_load1(uint32_t a[4], const uint32_t* rb, int mf, int tb, uint32_t toff,
                                         uint32_t tsh, int lane) {
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = k < mf ? ldg(rb + 32 * k + lane) : 0u;
  if (mf < 4) {
    const uint32_t t = pk_tail(rb, mf, tb, toff, tsh);
    a[0] = mf == 0 ? t : a[0];
    a[1] = mf == 1 ? t : a[1];
    a[2] = mf == 2 ? t : a[2];
    a[3] = mf == 3 ? t : a[3];
  }
}

// acc[i][r] += product row r of words x with v (the policy's arithmetic,
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

template <int EVAL, int POL>
__global__ void __launch_bounds__(32 * kPkWarps, 2) k_pk_gemv(PkTable T, unsigned long long* status) {
  using A = PkAcc<POL>;
  using AT = typename A::T;
  const uint64_t gband = blockIdx.x / kPkSplit;
  const int part = (int)(blockIdx.x % kPkSplit);
  if (gband >= T.total_bands) return;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint64_t first = 0;
  int jidx = -1;
  if (T.jobs != nullptr) {
    int lo = 0, hi = T.n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (T.prefix[mid] <= gband) lo = mid; else hi = mid - 1;
    }
    jidx = lo;
    first = T.prefix[jidx];
  }
  const PkJob& J = jidx < 0 ? T.single : T.jobs[jidx];
  const PkView P = J.p;
  const float* __restrict__ v = J.v;
  const float4* __restrict__ U = J.U;
  const uint64_t band = J.band0 + (gband - first);
  const int nrows = pk::band_rows(P.g, band);
  const uint64_t bc = P.g.bc;
  const bool v_aligned = ((reinterpret_cast<uintptr_t>(v) & 15u) == 0);
  const uint32_t last_colmask = (P.g.cols & 3) ? ((1u << (P.g.cols & 3)) - 1u) : 0xFu;

  __shared__ pk::FieldPar s_par[kPkWarps][16];
  __shared__ AT s_rs[kPkWarps][16];
  __shared__ pk::Seg s_seg[kPkWarps];
  pk::FieldPar* par = s_par[warp];
  AT* rs = s_rs[warp];
  if (lane < 16) rs[lane] = (AT)0;
  A acc;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc.v[i][r] = (AT)0;

  const int vw = part * kPkWarps + warp;
  for (uint64_t sb = vw; sb < P.g.nsegb; sb += kVW) {
    const pk::Seg S = P.segs[band * P.g.nsegb + sb];
    const int L = pk::seg_L(S), mf = L >> 5, tb = L & 31;
    const int We = pk::seg_We(S);
    const uint64_t TW = pk::tile_words(nrows, L);
    const int ntl = pk::seg_tiles(P.g, sb);
    const uint32_t ebase = (uint32_t)pk::seg_emax_base(S);
    const uint32_t ebase_bits = (ebase - 59u) << 23;   // binary32 2^(emax_base - 186)
    const uint32_t* sbody = P.body + S.body;
    if (!pk::seg_generic(S)) {
      __syncwarp();
      if (lane < 16) par[lane] = pk::field_param(S, lane);
      __syncwarp();
      const bool k2 = pk::seg_k2(S);
      // fields 3..8: w[0] bits 15..29 and w[1] bits 0..14; 9..15: w[1] bits
      // 15..29 and w[2] bits 0..19
      const bool hasA = ((S.w[0] >> 15) & 0x7FFFu) != 0 || (S.w[1] & 0x7FFFu) != 0;
      const bool hasB = ((S.w[1] >> 15) & 0x7FFFu) != 0 || (S.w[2] & 0xFFFFFu) != 0;
      const uint32_t tbit = (uint32_t)lane * (uint32_t)tb;
      const uint32_t toff = tbit >> 5, tsh = tbit & 31;
      for (int tt = 0; tt < ntl; ++tt) {
        const uint64_t col = (sb * pk::kSegTiles + tt) * pk::kTile + lane;
        const bool active = col < bc;
        const uint32_t* tbase = sbody + tt * TW;
        if (EVAL == WHFF_EVAL_COEFF) {
          uint32_t a[4][4];
          pk_load4(a, tbase, L, mf, tb, toff, tsh, lane);
          const float4 u4 = active ? ldg(U + col) : make_float4(0.f, 0.f, 0.f, 0.f);
          const float u[4] = {u4.x, u4.y, u4.z, u4.w};
          float w[4][4];
          const pk::FieldPar p0 = lds_par(par);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float f0 = __int2float_rn(pk::field_dc(a[i][0], a[i][1], p0));
            w[i][0] = __fmul_rn(f0, u[0]);
            w[i][1] = w[i][2] = w[i][3] = 0.0f;
          }
          // c = 1, 2: integer fields (up to 28 bits), binary32 by rounding
          auto field_int = [&](auto C, int k) {
            constexpr int c = decltype(C)::value;
            constexpr int r = seq_pos(c) >> 2, j = seq_pos(c) & 3;
            const pk::FieldPar p = lds_par(par + c);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t hi = k == 0 ? a[i][0] : a[i][1];
              const uint32_t lo = k == 0 ? a[i][1] : a[i][2];
              w[i][r] = __fmaf_rn(__int2float_rn(pk::field_i(hi, lo, p)), u[j], w[i][r]);
            }
          };
          auto field = [&](auto C, int k) {
            constexpr int c = decltype(C)::value;
            constexpr int r = seq_pos(c) >> 2, j = seq_pos(c) & 3;
            const pk::FieldPar p = lds_par(par + c);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t hi = k == 0 ? a[i][0] : k == 1 ? a[i][1] : a[i][2];
              const uint32_t lo = k == 0 ? a[i][1] : k == 1 ? a[i][2] : a[i][3];
              w[i][r] = __fmaf_rn(pk::field_f(hi, lo, p), u[j], w[i][r]);
            }
          };
          field_int(std::integral_constant<int, 1>(), 0);
          if (k2) field_int(std::integral_constant<int, 2>(), 1);
          else field_int(std::integral_constant<int, 2>(), 0);
          if (hasA) {
            field(std::integral_constant<int, 3>(), 1);
            field(std::integral_constant<int, 4>(), 1);
            field(std::integral_constant<int, 5>(), 1);
            field(std::integral_constant<int, 6>(), 1);
            field(std::integral_constant<int, 7>(), 1);
            field(std::integral_constant<int, 8>(), 1);
          }
          if (hasB) {
            field(std::integral_constant<int, 9>(), 2);
            field(std::integral_constant<int, 10>(), 2);
            field(std::integral_constant<int, 11>(), 2);
            field(std::integral_constant<int, 12>(), 2);
            field(std::integral_constant<int, 13>(), 2);
            field(std::integral_constant<int, 14>(), 2);
            field(std::integral_constant<int, 15>(), 2);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t e = pk::field_edelta(a[i][0], We);
            // (lanes past the row end: garbage records, scale 0)
            const float sc = active ? __uint_as_float(ebase_bits + (e << 23)) : 0.0f;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const float t = __fmul_rn(w[i][r], sc);
              if (POL == WHFF_POLICY_SINGLE) acc.v[i][r] = __fadd_rn(acc.v[i][r], t);
              else acc.v[i][r] = __dadd_rn(acc.v[i][r], (double)t);
            }
          }
        } else if (active) {
          // exact evaluation: the reference's words (bit-exact) x v
          const float4 v4 = load_v4(v, col, P.g.cols, v_aligned);
          const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
          const uint32_t colmask = (col + 1 == bc) ? last_colmask : 0xFu;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (i >= nrows) break;
            uint32_t ai[4];
            pk_load1(ai, tbase + i * L, mf, tb, toff, tsh, lane);
            int32_t q[16];
            pk_fields_int(ai, par, k2, q);
            float x[16];
            pk::words_from_q(q, ebase + pk::field_edelta(ai[0], We), x);
#pragma unroll
            for (int kk = 0; kk < 16; ++kk)
              if (!((colmask >> (kk & 3)) & 1u)) x[kk] = 0.0f;
            pk_acc_words<POL>(acc.v[i], x, vv);
          }
        }
      }
    } else {
      // generic segment: per-lane sequential parse of arbitrary records
      __syncwarp();
      if (lane == 0) s_seg[warp] = S;
      __syncwarp();
      for (int tt = 0; tt < ntl; ++tt) {
        const uint64_t col = (sb * pk::kSegTiles + tt) * pk::kTile + lane;
        if (col >= bc) continue;
        const float4 u4 = EVAL == WHFF_EVAL_COEFF ? ldg(U + col) : load_v4(v, col, P.g.cols, v_aligned);
        const float u[4] = {u4.x, u4.y, u4.z, u4.w};
        const uint32_t colmask = (col + 1 == bc) ? last_colmask : 0xFu;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i >= nrows) break;
          int32_t q[16];
          uint32_t ed;
#ifndef WHFF_NO_GENERIC
          pk_generic_parse(&s_seg[warp], sbody + tt * TW + (uint64_t)i * L, lane, q, &ed);
#else
          ed = 0; for (int c = 0; c < 16; ++c) q[c] = 0;
#endif
          if (EVAL == WHFF_EVAL_COEFF) {
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
              const float t = __fmul_rn(w[r], sc);
              if (POL == WHFF_POLICY_SINGLE) acc.v[i][r] = __fadd_rn(acc.v[i][r], t);
              else acc.v[i][r] = __dadd_rn(acc.v[i][r], (double)t);
            }
          } else {
            float x[16];
            pk::words_from_q(q, ebase + ed, x);
#pragma unroll
            for (int kk = 0; kk < 16; ++kk)
              if (!((colmask >> (kk & 3)) & 1u)) x[kk] = 0.0f;
            pk_acc_words<POL>(acc.v[i], x, u);
          }
        }
      }
    }
    if (S.exc_count) pk_exceptions<POL, AT>(P, v, band, S.exc_begin, S.exc_count, lane, rs);
  }

  // warp butterfly over the 16 rows, publish, last warp of the band combines
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc.v[i][r] = acc.v[i][r] + __shfl_xor_sync(0xFFFFFFFFu, acc.v[i][r], o);
  __syncwarp();
  PkRec* grec = T.recs + gband * kVW;
  unsigned last = 0;
  if (lane == 0) {
    PkRec& R = grec[vw];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (POL == WHFF_POLICY_SINGLE) {
          R.f[4 * i + r] = (float)acc.v[i][r];
          R.rf[4 * i + r] = (float)rs[4 * i + r];
        } else {
          R.d[4 * i + r] = (double)acc.v[i][r];
          R.r[4 * i + r] = (double)rs[4 * i + r];
        }
      }
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;"
                 : "=r"(old) : "l"(T.tickets + gband), "r"(kVW - 1u) : "memory");
    last = old == kVW - 1u;
  }
  if (!__shfl_sync(0xFFFFFFFFu, last, 0)) return;
  __syncwarp();
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  // lane = virtual warp: 32 records, fixed butterfly per row
  AT D[16], R[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    if (POL == WHFF_POLICY_SINGLE) {
      D[k] = (AT)__ldcg(&grec[lane].f[k]);
      R[k] = (AT)__ldcg(&grec[lane].rf[k]);
    } else {
      D[k] = (AT)__ldcg(&grec[lane].d[k]);
      R[k] = (AT)__ldcg(&grec[lane].r[k]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      D[k] = D[k] + __shfl_xor_sync(0xFFFFFFFFu, D[k], o);
      R[k] = R[k] + __shfl_xor_sync(0xFFFFFFFFu, R[k], o);
    }
  if (lane < 16) {
    const int i = lane >> 2, rr = lane & 3;
    const uint64_t row = (band * pk::kBand + i) * 4 + rr;
    if (i < nrows && row >= J.row_begin && row < J.row_end && row < P.g.rows) {
      float out;
      AT rsel = R[0], d0 = D[0], d1 = D[1], d2 = D[2], d3 = D[3], dsel = D[0];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k == lane) { rsel = R[k]; dsel = D[k]; }
        if (k == 4 * i + 0) d0 = D[k];
        if (k == 4 * i + 1) d1 = D[k];
        if (k == 4 * i + 2) d2 = D[k];
        if (k == 4 * i + 3) d3 = D[k];
      }
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
        if (POL == WHFF_POLICY_SINGLE) out = __fadd_rn((float)dsel, (float)rsel);
        else out = __double2float_rn(__dadd_rn((double)dsel, (double)rsel));
      }
      J.y[row - J.row_begin] = out;
      if (!isfinite(out)) atomicMin(status, (unsigned long long)row);
    }
  }
}

// ---------------------------------------------------------------------------
// fused decode + GEMV, coefficient evaluation, TMA-staged (the hot path)
// ---------------------------------------------------------------------------
// k_pk_gemv2 computes exactly what k_pk_gemv<COEFF> computes (same
// per-virtual-warp work, same operations in the same order per accumulator:
// bit-identical results) but is built for the B200's issue rate:
//   * every warp runs its own kP2Stages-deep ring of shared-memory stages;
//     lane 0 fills it with 1-D bulk copies (cp.async.bulk, the TMA engine)
//     of whole tiles (band x 32 block-columns of records, contiguous in HBM)
//     plus the tile's slice of U = G^T v, completing on a per-stage
//     mbarrier -- no registers are spent on loads in flight and the copies
//     of the next tiles overlap the decode of this one;
//   * the four block-rows of a band are decoded as two pairs with the
//     packed-f32x2 pipe ops (FADD2 for the magic-number conversion, FFMA2 for
//     the coefficient x u products, FMUL2 for the 2^k scales);
//   * segment headers of the warp's segments are read once into shared
//     memory.
// Generic segments (fields too wide for the fast path) and exceptions take
// the per-lane path of k_pk_gemv on global memory.
constexpr int kP2Warps = 4;                              // warps per CTA
constexpr int kP2Split = kPkVW / kP2Warps;               // CTAs per band
#ifndef WHFF_P2_STAGES
#define WHFF_P2_STAGES 4
#endif
#ifndef WHFF_P2_MINB
#define WHFF_P2_MINB 4
#endif
constexpr int kP2Stages = WHFF_P2_STAGES;                // power of two
static_assert((kP2Stages & (kP2Stages - 1)) == 0, "stage count must be a power of two");
constexpr int kP2TileWords = pk::kBand * 128;            // fast path: L <= 128
constexpr int kP2StageBytes = kP2TileWords * 4 + 32 * 16 + 128;   // tile + U slice + tail slack
constexpr int kP2HdrRing = 64;                           // segment headers held per warp (ring)

template <typename AT>
struct alignas(128) P2Warp {
  uint8_t stage[kP2Stages][kP2StageBytes];
  uint64_t bar[kP2Stages];
  pk::Seg seg[kP2HdrRing];
  pk::FieldPar par[16];
  float2 off2[16];     // (p.w, p.w) of every field as a float pair (FADD2 operand)
  AT rs[16];
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W2_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W2_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completing `bytes` on the stage's mbarrier
// (evict-first: the packed records are read once per launch)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

// Record words of one tile row from shared memory (as pk_load4's rows).
__device__ __forceinline__ void p2_row(uint32_t a[4], const uint32_t* rb, int mf, int tb, uint32_t toff,
                                       uint32_t tsh, int lane) {
  auto tail = [&](int m) -> uint32_t {
    if (!tb) return 0u;
    const uint32_t* q = rb + 32 * m + toff;
    return fsl(q[0], q[1], tsh);
  };
  switch (mf) {
    case 0: a[0] = tail(0); a[1] = a[2] = a[3] = 0u; break;
    case 1: a[0] = rb[lane]; a[1] = tail(1); a[2] = a[3] = 0u; break;
    case 2: a[0] = rb[lane]; a[1] = rb[32 + lane]; a[2] = tail(2); a[3] = 0u; break;
    case 3: a[0] = rb[lane]; a[1] = rb[32 + lane]; a[2] = rb[64 + lane]; a[3] = tail(3); break;
    default: a[0] = rb[lane]; a[1] = rb[32 + lane]; a[2] = rb[64 + lane]; a[3] = rb[96 + lane]; break;
  }
}

// ... the same with the record length's full-word count MF fixed at compile
// time (MF < 0: any, through p2_row)
template <int MF>
__device__ __forceinline__ void p2_row_t(uint32_t a[4], const uint32_t* rb, int mf, int tb, uint32_t toff,
                                         uint32_t tsh, int lane) {
  if constexpr (MF < 0) {
    p2_row(a, rb, mf, tb, toff, tsh, lane);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = k < MF ? rb[32 * k + lane] : 0u;
    if constexpr (MF < 4) {
      const uint32_t* q = rb + 32 * MF + toff;
      a[MF] = tb ? fsl(q[0], q[1], tsh) : 0u;
    }
  }
}

// The warp's pipeline cursor over the tiles of its fast segments.
struct P2Cursor {
  int k;    // index of the warp's segment (sb = vw + 32 k)
  int t;    // tile within it
};

template <int POL>
__global__ void __launch_bounds__(32 * kP2Warps, WHFF_P2_MINB) k_pk_gemv2(PkTable T, unsigned long long* status) {
  using A = PkAcc<POL>;
  using AT = typename A::T;
  extern __shared__ __align__(128) uint8_t p2_smem[];
  const uint64_t gband = blockIdx.x / kP2Split;
  const int part = (int)(blockIdx.x % kP2Split);
  if (gband >= T.total_bands) return;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  P2Warp<AT>& W = reinterpret_cast<P2Warp<AT>*>(p2_smem)[warp];
  uint64_t first = 0;
  int jidx = -1;
  if (T.jobs != nullptr) {
    int lo = 0, hi = T.n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (T.prefix[mid] <= gband) lo = mid; else hi = mid - 1;
    }
    jidx = lo;
    first = T.prefix[jidx];
  }
  const PkJob& J = jidx < 0 ? T.single : T.jobs[jidx];
  const PkView P = J.p;
  const float* __restrict__ v = J.v;
  const float4* __restrict__ U = J.U;
  const uint64_t band = J.band0 + (gband - first);
  const int nrows = pk::band_rows(P.g, band);
  const uint64_t bc = P.g.bc;
  const int vw = part * kP2Warps + warp;
  const int nseg = P.g.nsegb > (uint64_t)vw ? (int)((P.g.nsegb - 1 - vw) / kVW + 1) : 0;

  // segment headers -> a shared-memory ring, 32 at a time (the producer runs
  // at most kP2Stages tiles ahead of the consumer, so a header is never
  // overwritten while either still needs it)
  int hdr_loaded = 0;
  auto ensure_hdr = [&](int k) {
    while (k >= hdr_loaded) {
      __syncwarp();
      const int kk = hdr_loaded + lane;
      if (kk < nseg) W.seg[kk & (kP2HdrRing - 1)] = P.segs[band * P.g.nsegb + vw + (uint64_t)kVW * kk];
      hdr_loaded += 32;
      __syncwarp();
    }
  };
  auto hdr = [&](int k) -> const pk::Seg& { return W.seg[k & (kP2HdrRing - 1)]; };
  ensure_hdr(0);
  if (lane < 16) W.rs[lane] = (AT)0;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < kP2Stages; ++i) mbar_init(&W.bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));

  // producer (lane 0 issues; the cursor is warp-uniform)
  P2Cursor pc{0, 0};
  auto skip_generic = [&](P2Cursor& c) {
    while (c.k < nseg) {
      ensure_hdr(c.k);
      if (!pk::seg_generic(hdr(c.k)) && c.t < pk::seg_tiles(P.g, vw + (uint64_t)kVW * c.k)) break;
      ++c.k;
      c.t = 0;
    }
  };
  skip_generic(pc);
  uint32_t issued = 0;
  auto issue = [&]() {
    if (pc.k >= nseg) return;
    const uint64_t sb = vw + (uint64_t)kVW * pc.k;
    const pk::Seg& S = hdr(pc.k);
    const int L = pk::seg_L(S);
    const uint32_t tw = (uint32_t)pk::tile_words(nrows, L);
    const int slot = (int)(issued & (kP2Stages - 1));
    if (lane == 0) {
      const uint64_t col0 = (sb * pk::kSegTiles + pc.t) * pk::kTile;
      const uint32_t ubytes = (uint32_t)((bc - col0 < (uint64_t)pk::kTile ? bc - col0 : (uint64_t)pk::kTile) * 16);
      uint8_t* st = W.stage[slot];
      mbar_expect_tx(&W.bar[slot], tw * 4 + ubytes);
      bulk_g2s(st, P.body + S.body + (uint64_t)pc.t * tw, tw * 4, &W.bar[slot], policy);
      bulk_g2s(st + kP2TileWords * 4, U + col0, ubytes, &W.bar[slot], policy);
    }
    ++issued;
    ++pc.t;
    skip_generic(pc);
  };
  for (int i = 0; i < kP2Stages; ++i) issue();

  // Accumulators.  single: binary32 sums.  mixed: compensated binary32
  // pairs (s, c) per (block-row i, coefficient row r), kept as float2 over
  // the row pairs (0,1), (2,3) for the packed-f32x2 pipe; s + c goes to
  // binary64 once, before the warp butterfly (no per-block conversions).
  A acc;
  float2 ks[2][4], kc[2][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc.v[i][r] = (AT)0;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int r = 0; r < 4; ++r) ks[h][r] = kc[h][r] = make_float2(0.0f, 0.0f);
  // s' = s + t; c += (s - s') + t
  auto kahan2 = [](float2& S, float2& C, float2 t) {
    const float2 s1 = __fadd2_rn(S, t);
    const float2 d = __fadd2_rn(S, make_float2(-s1.x, -s1.y));
    C = __fadd2_rn(C, __fadd2_rn(d, t));
    S = s1;
  };
  uint32_t consumed = 0;
  const uint32_t last_colmask = (P.g.cols & 3) ? ((1u << (P.g.cols & 3)) - 1u) : 0xFu;
  const bool v_aligned = ((reinterpret_cast<uintptr_t>(v) & 15u) == 0);

  for (int k = 0; k < nseg; ++k) {
    const uint64_t sb = vw + (uint64_t)kVW * k;
    ensure_hdr(k);
    const pk::Seg S = hdr(k);
    const int L = pk::seg_L(S), mf = L >> 5, tb = L & 31;
    const int We = pk::seg_We(S);
    const int ntl = pk::seg_tiles(P.g, sb);
    const uint32_t ebase = (uint32_t)pk::seg_emax_base(S);
    const uint32_t ebase_bits = (ebase - 59u) << 23;   // binary32 2^(emax_base - 186)
    if (!pk::seg_generic(S)) {
      __syncwarp();
      if (lane < 16) {
        const pk::FieldPar fp = pk::field_param(S, lane);
        W.par[lane] = fp;
        W.off2[lane] = make_float2(__uint_as_float(fp.w), __uint_as_float(fp.w));
      }
      __syncwarp();
      const bool k2 = pk::seg_k2(S);
      const bool hasA = ((S.w[0] >> 15) & 0x7FFFu) != 0 || (S.w[1] & 0x7FFFu) != 0;
      const bool hasB = ((S.w[1] >> 15) & 0x7FFFu) != 0 || (S.w[2] & 0xFFFFFu) != 0;
      const uint32_t tbit = (uint32_t)lane * (uint32_t)tb;
      const uint32_t toff = tbit >> 5, tsh = tbit & 31;
      auto tiles = [&](auto MFC) {
      constexpr int MF = decltype(MFC)::value;
      for (int tt = 0; tt < ntl; ++tt) {
        const int slot = (int)(consumed & (kP2Stages - 1));
        mbar_wait(&W.bar[slot], (consumed / kP2Stages) & 1u);
        const uint64_t col = (sb * pk::kSegTiles + tt) * pk::kTile + lane;
        const bool active = col < bc;
        const uint32_t* tbase = reinterpret_cast<const uint32_t*>(W.stage[slot]);
        const float4 u4 = active ? reinterpret_cast<const float4*>(W.stage[slot] + kP2TileWords * 4)[lane]
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        const float2 uu[4] = {make_float2(u4.x, u4.x), make_float2(u4.y, u4.y), make_float2(u4.z, u4.z),
                              make_float2(u4.w, u4.w)};
        uint32_t a[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) p2_row_t<MF>(a[i], tbase + i * L, mf, tb, toff, tsh, lane);
        // w[pair][r] = (w[2 pair][r], w[2 pair + 1][r])
        float2 w[2][4];
        {
          const pk::FieldPar p0 = lds_par(&W.par[0]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float f0a = __int2float_rn(pk::field_dc(a[2 * h][0], a[2 * h][1], p0));
            const float f0b = __int2float_rn(pk::field_dc(a[2 * h + 1][0], a[2 * h + 1][1], p0));
            w[h][0] = __fmul2_rn(make_float2(f0a, f0b), uu[0]);
            w[h][1] = w[h][2] = w[h][3] = make_float2(0.0f, 0.0f);
          }
        }
        auto field_int = [&](auto C, int kk) {
          constexpr int c = decltype(C)::value;
          constexpr int r = seq_pos(c) >> 2, j = seq_pos(c) & 3;
          const pk::FieldPar p = lds_par(&W.par[c]);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t hia = kk == 0 ? a[2 * h][0] : a[2 * h][1];
            const uint32_t loa = kk == 0 ? a[2 * h][1] : a[2 * h][2];
            const uint32_t hib = kk == 0 ? a[2 * h + 1][0] : a[2 * h + 1][1];
            const uint32_t lob = kk == 0 ? a[2 * h + 1][1] : a[2 * h + 1][2];
            const float2 q = make_float2(__int2float_rn(pk::field_i(hia, loa, p)),
                                         __int2float_rn(pk::field_i(hib, lob, p)));
            w[h][r] = __ffma2_rn(q, uu[j], w[h][r]);
          }
        };
        auto field = [&](auto C, int kk) {
          constexpr int c = decltype(C)::value;
          constexpr int r = seq_pos(c) >> 2, j = seq_pos(c) & 3;
          const pk::FieldPar p = lds_par(&W.par[c]);
          const float2 o2 = W.off2[c];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t hia = kk == 0 ? a[2 * h][0] : kk == 1 ? a[2 * h][1] : a[2 * h][2];
            const uint32_t loa = kk == 0 ? a[2 * h][1] : kk == 1 ? a[2 * h][2] : a[2 * h][3];
            const uint32_t hib = kk == 0 ? a[2 * h + 1][0] : kk == 1 ? a[2 * h + 1][1] : a[2 * h + 1][2];
            const uint32_t lob = kk == 0 ? a[2 * h + 1][1] : kk == 1 ? a[2 * h + 1][2] : a[2 * h + 1][3];
            const uint32_t fa = fsr(pk::fsl64(hia, loa, p.x), p.y, p.z);
            const uint32_t fb = fsr(pk::fsl64(hib, lob, p.x), p.y, p.z);
            const float2 q = __fadd2_rn(make_float2(__uint_as_float(fa), __uint_as_float(fb)), o2);
            w[h][r] = __ffma2_rn(q, uu[j], w[h][r]);
          }
        };
        field_int(std::integral_constant<int, 1>(), 0);
        if (k2) field_int(std::integral_constant<int, 2>(), 1);
        else field_int(std::integral_constant<int, 2>(), 0);
        if (hasA) {
          field(std::integral_constant<int, 3>(), 1);
          field(std::integral_constant<int, 4>(), 1);
          field(std::integral_constant<int, 5>(), 1);
          field(std::integral_constant<int, 6>(), 1);
          field(std::integral_constant<int, 7>(), 1);
          field(std::integral_constant<int, 8>(), 1);
        }
        if (hasB) {
          field(std::integral_constant<int, 9>(), 2);
          field(std::integral_constant<int, 10>(), 2);
          field(std::integral_constant<int, 11>(), 2);
          field(std::integral_constant<int, 12>(), 2);
          field(std::integral_constant<int, 13>(), 2);
          field(std::integral_constant<int, 14>(), 2);
          field(std::integral_constant<int, 15>(), 2);
        }
        // all lanes are done with the stage: refill it with the tile kP2Stages ahead
        __syncwarp();
        ++consumed;
        issue();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t ea = pk::field_edelta(a[2 * h][0], We), eb = pk::field_edelta(a[2 * h + 1][0], We);
          // (lanes past the row end: scale 0)
          const float2 sc = active ? make_float2(__uint_as_float(ebase_bits + (ea << 23)),
                                                 __uint_as_float(ebase_bits + (eb << 23)))
                                   : make_float2(0.0f, 0.0f);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const float2 t = __fmul2_rn(w[h][r], sc);
            if (POL == WHFF_POLICY_SINGLE) {
              acc.v[2 * h][r] = __fadd_rn(acc.v[2 * h][r], t.x);
              acc.v[2 * h + 1][r] = __fadd_rn(acc.v[2 * h + 1][r], t.y);
            } else {
              kahan2(ks[h][r], kc[h][r], t);
            }
          }
        }
      }
      };
#ifdef WHFF_P2_MF_TEMPLATES
      if (mf == 2) tiles(std::integral_constant<int, 2>());
      else if (mf == 3) tiles(std::integral_constant<int, 3>());
      else
#endif
      tiles(std::integral_constant<int, -1>());
    } else {
      // generic segment (not staged): per-lane sequential parse from global memory
      const uint64_t TW = pk::tile_words(nrows, L);
      const uint32_t* sbody = P.body + S.body;
      for (int tt = 0; tt < ntl; ++tt) {
        const uint64_t col = (sb * pk::kSegTiles + tt) * pk::kTile + lane;
        if (col >= bc) continue;
        const float4 u4 = ldg(U + col);
        const float u[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i >= nrows) break;
          int32_t q[16];
          uint32_t ed;
#ifndef WHFF_NO_GENERIC
          pk_generic_parse(&hdr(k), sbody + tt * TW + (uint64_t)i * L, lane, q, &ed);
#else
          ed = 0; for (int c = 0; c < 16; ++c) q[c] = 0;
#endif
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
            const float t = __fmul_rn(w[r], sc);
            if (POL == WHFF_POLICY_SINGLE) acc.v[i][r] = __fadd_rn(acc.v[i][r], t);
            else kahan2(ks[i >> 1][r], kc[i >> 1][r], (i & 1) ? make_float2(0.0f, t) : make_float2(t, 0.0f));
          }
        }
      }
      (void)last_colmask;
      (void)v_aligned;
    }
    if (S.exc_count) pk_exceptions<POL, AT>(P, v, band, S.exc_begin, S.exc_count, lane, W.rs);
  }

  if (POL != WHFF_POLICY_SINGLE) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        acc.v[2 * h][r] = __dadd_rn((double)ks[h][r].x, (double)kc[h][r].x);
        acc.v[2 * h + 1][r] = __dadd_rn((double)ks[h][r].y, (double)kc[h][r].y);
      }
  }

  // warp butterfly over the 16 rows, publish, last warp of the band combines
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc.v[i][r] = acc.v[i][r] + __shfl_xor_sync(0xFFFFFFFFu, acc.v[i][r], o);
  __syncwarp();
  PkRec* grec = T.recs + gband * kVW;
  unsigned last = 0;
  if (lane == 0) {
    PkRec& R = grec[vw];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (POL == WHFF_POLICY_SINGLE) {
          R.f[4 * i + r] = (float)acc.v[i][r];
          R.rf[4 * i + r] = (float)W.rs[4 * i + r];
        } else {
          R.d[4 * i + r] = (double)acc.v[i][r];
          R.r[4 * i + r] = (double)W.rs[4 * i + r];
        }
      }
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;"
                 : "=r"(old) : "l"(T.tickets + gband), "r"(kVW - 1u) : "memory");
    last = old == kVW - 1u;
  }
  if (!__shfl_sync(0xFFFFFFFFu, last, 0)) return;
  __syncwarp();
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  AT D[16], R[16];
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    if (POL == WHFF_POLICY_SINGLE) {
      D[kk] = (AT)__ldcg(&grec[lane].f[kk]);
      R[kk] = (AT)__ldcg(&grec[lane].rf[kk]);
    } else {
      D[kk] = (AT)__ldcg(&grec[lane].d[kk]);
      R[kk] = (AT)__ldcg(&grec[lane].r[kk]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      D[kk] = D[kk] + __shfl_xor_sync(0xFFFFFFFFu, D[kk], o);
      R[kk] = R[kk] + __shfl_xor_sync(0xFFFFFFFFu, R[kk], o);
    }
  if (lane < 16) {
    const int i = lane >> 2, rr = lane & 3;
    const uint64_t row = (band * pk::kBand + i) * 4 + rr;
    if (i < nrows && row >= J.row_begin && row < J.row_end && row < P.g.rows) {
      float out;
      AT rsel = R[0], d0 = D[0], d1 = D[1], d2 = D[2], d3 = D[3];
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        if (kk == lane) rsel = R[kk];
        if (kk == 4 * i + 0) d0 = D[kk];
        if (kk == 4 * i + 1) d1 = D[kk];
        if (kk == 4 * i + 2) d2 = D[kk];
        if (kk == 4 * i + 3) d3 = D[kk];
      }
      const AT dd[4] = {d0, d1, d2, d3};
      if (POL == WHFF_POLICY_SINGLE) {
        float t = (float)rsel;
#pragma unroll
        for (int a2 = 0; a2 < 4; ++a2) t = __fmaf_rn(c_G[rr][a2], (float)dd[a2], t);
        out = t;
      } else {
        double t = (double)rsel;
#pragma unroll
        for (int a2 = 0; a2 < 4; ++a2) t = __fma_rn((double)c_G[rr][a2], (double)dd[a2], t);
        out = __double2float_rn(t);
      }
      J.y[row - J.row_begin] = out;
      if (!isfinite(out)) atomicMin(status, (unsigned long long)row);
    }
  }
}



template <int POL>
static cudaError_t p2_launch(const PkTable& T, unsigned long long* status, cudaStream_t cs) {
  using AT = typename PkAcc<POL>::T;
  const size_t smem = sizeof(P2Warp<AT>) * kP2Warps;
  static bool attr = false;   // set once per process (the attribute is per function)
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_pk_gemv2<POL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const unsigned blocks = (unsigned)(T.total_bands * kP2Split);
  k_pk_gemv2<POL><<<blocks, 32 * kP2Warps, smem, cs>>>(T, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// decode-only (codec.decompress) from the packed layout: bit-exact words
// ---------------------------------------------------------------------------
// One warp per tile (band x 32 block-columns); exceptions are written by
// k_pk_exc_words afterwards (their records decode to zeros here).
__global__ void __launch_bounds__(256) k_pk_words(PkView P, float* out, uint64_t ld) {
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  if (wid >= P.g.nband * P.g.ntile) return;
  const uint64_t band = wid / P.g.ntile, t = wid % P.g.ntile;
  const uint64_t sb = t / pk::kSegTiles;
  const int tt = (int)(t % pk::kSegTiles);
  const int nrows = pk::band_rows(P.g, band);
  const pk::Seg S = P.segs[band * P.g.nsegb + sb];
  const int L = pk::seg_L(S), mf = L >> 5, tb = L & 31, We = pk::seg_We(S);
  const uint32_t ebase = (uint32_t)pk::seg_emax_base(S);
  const uint64_t TW = pk::tile_words(nrows, L);
  const uint64_t col = t * pk::kTile + lane;
  const bool active = col < P.g.bc;
  const uint32_t* base = P.body + S.body + tt * TW;
  __shared__ pk::FieldPar s_par[8][16];
  if (!pk::seg_generic(S)) {
    if (lane < 16) s_par[warp][lane] = pk::field_param(S, lane);
    __syncwarp();
  }
  if (!active) return;
  const bool vec = ((reinterpret_cast<uintptr_t>(out) | (ld * 4)) & 15u) == 0;
  uint32_t a[4][4];
  if (!pk::seg_generic(S)) {
    const uint32_t tbit = (uint32_t)lane * (uint32_t)tb;
    pk_load4(a, base, L, mf, tb, tbit >> 5, tbit & 31, lane);
  }
  int W[16];
  pk::Layout f;
  if (pk::seg_generic(S)) seg_layout(S, W, f);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i >= nrows) break;
    int32_t q[16];
    uint32_t ed;
    if (!pk::seg_generic(S)) {
      pk_fields_int(a[i], s_par[warp], pk::seg_k2(S), q);
      ed = pk::field_edelta(a[i][0], We);
    } else {
      uint32_t rec[pk::kMaxRecordWords + 1];
      pk_generic_record(base + (uint64_t)i * L, L, lane, rec);
      pk::parse_record(f, W, rec, ed, q);
    }
    float x[16];
    pk::words_from_q(q, ebase + ed, x);
    const uint64_t r0 = (band * pk::kBand + i) * 4, c0 = col * 4;
    if (vec && r0 + 4 <= P.g.rows && c0 + 4 <= P.g.cols) {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
        *reinterpret_cast<float4*>(out + (r0 + rr) * ld + c0) =
            make_float4(x[4 * rr], x[4 * rr + 1], x[4 * rr + 2], x[4 * rr + 3]);
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

template <int EVAL>
static void pk_gemv_pol(int policy, const PkTable& T, unsigned long long* status, cudaStream_t cs) {
  const unsigned blocks = (unsigned)(T.total_bands * kPkSplit);
  const unsigned threads = 32 * kPkWarps;
  if (policy == WHFF_POLICY_SINGLE) k_pk_gemv<EVAL, WHFF_POLICY_SINGLE><<<blocks, threads, 0, cs>>>(T, status);
  else if (EVAL == WHFF_EVAL_COEFF || policy == WHFF_POLICY_MIXED)
    k_pk_gemv<EVAL, WHFF_POLICY_MIXED><<<blocks, threads, 0, cs>>>(T, status);
  else
    k_pk_gemv<EVAL, (EVAL == WHFF_EVAL_COEFF ? WHFF_POLICY_MIXED : WHFF_POLICY_DOUBLE)>
        <<<blocks, threads, 0, cs>>>(T, status);
}

cudaError_t pk_launch_gemv(int eval, int policy, const PkTable& T, unsigned long long* status,
                           cudaStream_t cs) {
  if (T.total_bands == 0) return cudaSuccess;
  if (eval == WHFF_EVAL_COEFF) {
    if (policy == WHFF_POLICY_SINGLE) return p2_launch<WHFF_POLICY_SINGLE>(T, status, cs);
    return p2_launch<WHFF_POLICY_MIXED>(T, status, cs);
  }
  pk_gemv_pol<WHFF_EVAL_EXACT>(policy, T, status, cs);
  return cudaGetLastError();
}
