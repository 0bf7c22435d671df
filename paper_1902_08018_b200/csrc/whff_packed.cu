// whff_packed.cu -- kernels of the tile-packed layout (whff_packed.cuh):
// the packer (reference / skeleton-first stream -> packed), the fused
// decode + GEMV that reads it (the hot path), decode-only words, and the
// exception side list, and their host launchers (whff_packed_api.h).
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
  if (eval == WHFF_EVAL_COEFF) pk_gemv_pol<WHFF_EVAL_COEFF>(policy, T, status, cs);
  else pk_gemv_pol<WHFF_EVAL_EXACT>(policy, T, status, cs);
  return cudaGetLastError();
}
