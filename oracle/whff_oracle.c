/*
 * whff_oracle.c -- CPU restatement of the reference WHFF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels; it is linked/loaded only by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg.  The product package never imports it.
 *
 * Every function restates a reference function; citations are
 * file:line into /root/reference/pkg/src/whff/ (K = _kernels.pyx,
 * KP = _kernels_py.py, codec = codec.py, thermal = thermal.py).
 * Parity is pinned by tests/test_oracle.py against golden vectors produced
 * by the reference itself (tools/make_golden.py) and, when oracle/_ref is
 * built, against the live reference.
 *
 * Build: oracle/Makefile  (gcc -O2 -fno-fast-math -ffp-contract=off, so
 * binary32/binary64 rounding matches the Cython/numpy reference exactly).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_BLOCK 4        /* codec:27 */
#define ORC_N_PLANES 27    /* codec:28 */
#define ORC_QUANT_BITS 26  /* codec:29 */
#define ORC_EMAX_BIAS 160  /* codec:30 */

/* codec:40  total-sequency order, ties broken by row */
static const int SEQUENCY[16] = {0, 1, 4, 2, 5, 8, 3, 6, 9, 12, 7, 10, 13, 11, 14, 15};

int orc_sequency(int i) { return SEQUENCY[i]; }

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* np.unpackbits is MSB-first within each byte (K:374-375). */
static inline int getbit(const uint8_t* p, int64_t pos) {
    return (p[pos >> 3] >> (7 - (pos & 7))) & 1;
}

/* ------------------------------------------------------------------------ */
/* decode: K:286-368 (_decode_one), K:371-408 (decode_blocks)               */
/* ------------------------------------------------------------------------ */
static int64_t decode_one(const uint8_t* bits, int64_t start, int64_t limit,
                          uint32_t* mag, uint8_t* neg, uint32_t* raw_words,
                          uint16_t* emax_out, uint8_t* raw_out, int n_planes,
                          int planes_limit, int has_raw_flag) {
    int64_t pos = start;
    int code = 0, i, p, c, v, flag, hit, s, nrem, k, rem_start;
    uint32_t w;
    unsigned char sig[16];
    int remaining[16];

    for (i = 0; i < 9; i++) {
        if (pos >= limit) return pos;
        code = (code << 1) | getbit(bits, pos);
        pos++;
    }
    *emax_out = (uint16_t)code;
    if (has_raw_flag) {
        if (pos >= limit) return pos;
        v = getbit(bits, pos);
        pos++;
        if (v) {
            *raw_out = 1;
            for (c = 0; c < 16; c++) {
                w = 0;
                for (i = 0; i < 32; i++) {
                    if (pos >= limit) return pos;
                    w = (w << 1) | (uint32_t)getbit(bits, pos);
                    pos++;
                }
                raw_words[c] = w;
            }
            return pos;
        }
    }
    if (code == 0) return pos;
    for (c = 0; c < 16; c++) sig[c] = 0;
    for (p = n_planes - 1; p > n_planes - 1 - planes_limit; p--) {
        if (pos >= limit) break;
        for (c = 0; c < 16; c++) {       /* refinement pass, index order */
            if (sig[c]) {
                if (pos >= limit) return pos;
                if (getbit(bits, pos)) mag[c] |= (uint32_t)1 << p;
                pos++;
            }
        }
        nrem = 0;                        /* significance pass */
        for (c = 0; c < 16; c++)
            if (!sig[c]) remaining[nrem++] = c;
        while (nrem > 0) {
            if (pos >= limit) return pos;
            flag = getbit(bits, pos);
            pos++;
            if (!flag) break;
            hit = 0;
            for (k = 0; k < nrem; k++) {
                c = remaining[k];
                if (pos >= limit) return pos;
                v = getbit(bits, pos);
                pos++;
                if (v) {
                    if (pos >= limit) return pos; /* sign unavailable: ignore hit */
                    s = getbit(bits, pos);
                    pos++;
                    mag[c] |= (uint32_t)1 << p;
                    neg[c] = (uint8_t)s;
                    sig[c] = 1;
                    rem_start = k + 1;     /* drop the consumed prefix (K:360-363) */
                    for (i = 0; i < nrem - rem_start; i++)
                        remaining[i] = remaining[rem_start + i];
                    nrem -= rem_start;
                    hit = 1;
                    break;
                }
            }
            if (!hit) break;
        }
    }
    return pos;
}

/* K:371-408.  Outputs must be zero-initialised by the caller (np.zeros). */
void orc_decode_blocks(const uint8_t* payload, int64_t payload_bytes,
                       const uint64_t* offsets, const uint64_t* seglens,
                       int64_t nb, int n_planes, int planes_limit,
                       int has_raw_flag, uint32_t* mag, uint8_t* neg,
                       uint16_t* emax_code, uint8_t* raw, uint32_t* raw_words,
                       uint64_t* consumed) {
    int64_t nbits = payload_bytes * 8;
    int64_t b;
#pragma omp parallel for schedule(static)
    for (b = 0; b < nb; b++) {
        int64_t start = (int64_t)offsets[b];
        int64_t limit = start + (int64_t)seglens[b];
        if (limit > nbits) limit = nbits;
        int64_t pos = decode_one(payload, start, limit, mag + 16 * b, neg + 16 * b,
                                 raw_words + 16 * b, emax_code + b, raw + b,
                                 n_planes, planes_limit, has_raw_flag);
        consumed[b] = (uint64_t)(pos - start);
    }
}

/* ------------------------------------------------------------------------ */
/* reconstruct: codec:128-134 (_inv_lift), :145-150 (_inverse_transform),   */
/* :201-206 (_dequantize), :209-218 (_reconstruct_blocks)                   */
/* ------------------------------------------------------------------------ */
static inline void inv_lift(int64_t* x, int64_t* y, int64_t* z, int64_t* w) {
    *y += *w >> 1; *w -= *y >> 1;
    *y += *w; *w *= 2; *w -= *y;
    *z += *x; *x *= 2; *x -= *z;
    *y += *z; *z *= 2; *z -= *y;
    *w += *x; *x *= 2; *x -= *w;
}

static inline void fwd_lift(int64_t* x, int64_t* y, int64_t* z, int64_t* w) {
    /* codec:118-125 */
    *x += *w; *x >>= 1; *w -= *x;
    *z += *y; *z >>= 1; *y -= *z;
    *x += *z; *x >>= 1; *z -= *x;
    *w += *y; *w >>= 1; *y -= *w;
    *w += *y >> 1; *y -= *w >> 1;
}

/* Integer coefficients (sequency order, signed) -> 4x4 raster q. */
static void inverse_transform(const int64_t* coef_seq, int64_t* q) {
    int64_t t[16];
    int i;
    for (i = 0; i < 16; i++) t[SEQUENCY[i]] = coef_seq[i]; /* [:, _INV_SEQUENCY] */
    for (i = 0; i < 4; i++)   /* columns first (swapaxes, lift) */
        inv_lift(&t[0 * 4 + i], &t[1 * 4 + i], &t[2 * 4 + i], &t[3 * 4 + i]);
    for (i = 0; i < 4; i++)   /* then rows */
        inv_lift(&t[i * 4 + 0], &t[i * 4 + 1], &t[i * 4 + 2], &t[i * 4 + 3]);
    memcpy(q, t, sizeof(t));
}

static void reconstruct_one(const uint32_t* mag, const uint8_t* neg,
                            uint16_t emax_code, uint8_t raw,
                            const uint32_t* raw_words, float* out) {
    int i;
    if (raw) {
        memcpy(out, raw_words, 16 * sizeof(float));
        return;
    }
    int64_t coef[16], q[16];
    for (i = 0; i < 16; i++) {
        coef[i] = (int64_t)mag[i];
        if (neg[i]) coef[i] = -coef[i];
    }
    inverse_transform(coef, q);
    int emax = (int)emax_code - ORC_EMAX_BIAS;
    double scale = ldexp(1.0, emax - ORC_QUANT_BITS);
    for (i = 0; i < 16; i++) {
        double d = emax_code == 0 ? 0.0 : (double)q[i] * scale;
        out[i] = (float)d;
    }
}

void orc_reconstruct_blocks(const uint32_t* mag, const uint8_t* neg,
                            const uint16_t* emax_code, const uint8_t* raw,
                            const uint32_t* raw_words, int64_t nb, float* out) {
    int64_t b;
#pragma omp parallel for schedule(static)
    for (b = 0; b < nb; b++)
        reconstruct_one(mag + 16 * b, neg + 16 * b, emax_code[b],
                        raw ? raw[b] : 0, raw_words + 16 * b, out + 16 * b);
}

/* codec:167-171: blocks (nb,4,4) in row-major block grid -> cropped array */
void orc_from_blocks(const float* blocks, int64_t rows, int64_t cols, float* out) {
    int64_t bc = (cols + 3) / 4;
    int64_t r;
#pragma omp parallel for schedule(static)
    for (r = 0; r < rows; r++) {
        for (int64_t c = 0; c < cols; c++) {
            int64_t b = (r / 4) * bc + c / 4;
            out[r * cols + c] = blocks[16 * b + 4 * (r % 4) + (c % 4)];
        }
    }
}

/* codec:296-314 minus validation (done in python): full decompress into
 * out[rows*cols]; returns index of first non-finite value or -1.        */
int64_t orc_decompress(const uint8_t* payload, int64_t payload_bytes,
                       const uint64_t* offsets, const uint64_t* seglens,
                       int64_t rows, int64_t cols, int planes_limit,
                       int has_raw_flag, float* out) {
    int64_t br = (rows + 3) / 4, bc = (cols + 3) / 4, nb = br * bc;
    int64_t nbits = payload_bytes * 8;
    int64_t first_bad = -1;
    int64_t brow;
#pragma omp parallel for schedule(dynamic, 1)
    for (brow = 0; brow < br; brow++) {
        uint32_t mag[16], rw[16];
        uint8_t neg[16], raw;
        uint16_t emax;
        float blk[16];
        for (int64_t bcol = 0; bcol < bc; bcol++) {
            int64_t b = brow * bc + bcol;
            memset(mag, 0, sizeof(mag));
            memset(rw, 0, sizeof(rw));
            memset(neg, 0, sizeof(neg));
            raw = 0;
            emax = 0;
            int64_t start = (int64_t)offsets[b];
            int64_t limit = start + (int64_t)seglens[b];
            if (limit > nbits) limit = nbits;
            decode_one(payload, start, limit, mag, neg, rw, &emax, &raw,
                       ORC_N_PLANES, planes_limit, has_raw_flag);
            reconstruct_one(mag, neg, emax, raw, rw, blk);
            for (int i = 0; i < 4; i++) {
                int64_t r = brow * 4 + i;
                if (r >= rows) break;
                for (int j = 0; j < 4; j++) {
                    int64_t c = bcol * 4 + j;
                    if (c >= cols) break;
                    out[r * cols + c] = blk[4 * i + j];
                }
            }
        }
    }
    (void)nb;
    for (int64_t i = 0; i < rows * cols; i++) {
        if (!isfinite(out[i])) { first_bad = i; break; }
    }
    return first_bad;
}

/* ------------------------------------------------------------------------ */
/* GEMV: K:24-47 (_seq_rows), K:50-77 (_tree_row_*), K:80-132 (gemv_kernel) */
/* policy 0 = mixed, 1 = single, 2 = double; shape 0 = sequential, 1 = tree */
/* ------------------------------------------------------------------------ */
static void tree_row_f64(double* buf, int64_t w, int fanout) {
    while (w > 1) {
        int64_t ngroups = (w + fanout - 1) / fanout;
        for (int64_t g = 0; g < ngroups; g++) {
            double acc = buf[g * fanout];
            for (int j = 1; j < fanout; j++) {
                int64_t idx = g * fanout + j;
                acc = acc + (idx < w ? buf[idx] : 0.0);
            }
            buf[g] = acc;
        }
        w = ngroups;
    }
}

static void tree_row_f32(float* buf, int64_t w, int fanout) {
    while (w > 1) {
        int64_t ngroups = (w + fanout - 1) / fanout;
        for (int64_t g = 0; g < ngroups; g++) {
            float acc = buf[g * fanout];
            for (int j = 1; j < fanout; j++) {
                int64_t idx = g * fanout + j;
                acc = acc + (idx < w ? buf[idx] : 0.0f);
            }
            buf[g] = acc;
        }
        w = ngroups;
    }
}

int orc_gemv(const float* m, const float* v, int64_t h, int64_t w, int policy,
             int shape, int fanout, float* out) {
    int64_t i;
    int err = 0;
    if (shape == 0) {
#pragma omp parallel for schedule(static)
        for (i = 0; i < h; i++) {
            const float* row = m + i * w;
            if (policy == 1) {
                float acc_f = 0.0f;
                for (int64_t j = 0; j < w; j++) {
                    float prod_f = row[j] * v[j];
                    acc_f = acc_f + prod_f;
                }
                out[i] = acc_f;
            } else if (policy == 2) {
                double acc_d = 0.0;
                for (int64_t j = 0; j < w; j++)
                    acc_d = acc_d + (double)row[j] * (double)v[j];
                out[i] = (float)acc_d;
            } else {
                double acc_d = 0.0;
                for (int64_t j = 0; j < w; j++) {
                    float prod_f = row[j] * v[j];
                    acc_d = acc_d + (double)prod_f;
                }
                out[i] = (float)acc_d;
            }
        }
        return 0;
    }
#pragma omp parallel
    {
        double* dbuf = NULL;
        float* fbuf = NULL;
        if (policy == 1) fbuf = (float*)malloc((size_t)w * sizeof(float));
        else dbuf = (double*)malloc((size_t)w * sizeof(double));
        if (!dbuf && !fbuf) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(static)
            for (i = 0; i < h; i++) {
                const float* row = m + i * w;
                if (policy == 1) {
                    for (int64_t j = 0; j < w; j++) fbuf[j] = row[j] * v[j];
                    tree_row_f32(fbuf, w, fanout);
                    out[i] = fbuf[0];
                } else {
                    if (policy == 2)
                        for (int64_t j = 0; j < w; j++) dbuf[j] = (double)row[j] * (double)v[j];
                    else
                        for (int64_t j = 0; j < w; j++) dbuf[j] = (double)(row[j] * v[j]);
                    tree_row_f64(dbuf, w, fanout);
                    out[i] = (float)dbuf[0];
                }
            }
        }
        free(dbuf);
        free(fbuf);
    }
    return err;
}

/* ------------------------------------------------------------------------ */
/* encode: codec:157-164 (_to_blocks), :186-198 (exponent, quantize),        */
/* :137-142 (_forward_transform), :225-268 (compress), :271-293             */
/* (_select_planes), K:139-225 (_encode_one), K:228-283 (encode_blocks)      */
/* ------------------------------------------------------------------------ */
#define ORC_MAX_BLOCK_BITS (9 + 1 + 16 * 32 + ORC_N_PLANES * (16 + 33))

/* Emits one block into `out` (one byte per bit); returns emitted length. */
static int encode_one(const int64_t* mag, const uint8_t* neg, int emax_code,
                      int planes, int raw, const uint32_t* raw_words,
                      int n_planes, int budget, int has_raw_flag, uint8_t* out) {
    int n = 0, i, p, c, bit, flag, hit, done, rem_start, nrem, k;
    unsigned char sig[16];
    int remaining[16];
    for (i = 8; i >= 0; i--) out[n++] = (emax_code >> i) & 1;
    if (has_raw_flag) out[n++] = raw ? 1 : 0;
    if (raw) {
        for (c = 0; c < 16; c++)
            for (i = 31; i >= 0; i--) out[n++] = (raw_words[c] >> i) & 1;
    } else if (emax_code != 0) {
        for (c = 0; c < 16; c++) sig[c] = 0;
        done = 0;
        for (p = n_planes - 1; p > n_planes - 1 - planes; p--) {
            if (done) break;
            for (c = 0; c < 16; c++) {
                if (sig[c]) {
                    if (budget && n >= budget) { done = 1; break; }
                    out[n++] = (mag[c] >> p) & 1;
                }
            }
            if (done) break;
            nrem = 0;
            for (c = 0; c < 16; c++)
                if (!sig[c]) remaining[nrem++] = c;
            while (nrem > 0) {
                if (budget && n >= budget) { done = 1; break; }
                flag = 0;
                for (k = 0; k < nrem; k++)
                    if ((mag[remaining[k]] >> p) & 1) { flag = 1; break; }
                out[n++] = (uint8_t)flag;
                if (!flag) break;
                hit = 0;
                for (k = 0; k < nrem; k++) {
                    c = remaining[k];
                    if (budget && n >= budget) { done = 1; break; }
                    bit = (mag[c] >> p) & 1;
                    if (bit && budget && n == budget - 1) {
                        out[n++] = 0; /* sign would not fit */
                        done = 1;
                        break;
                    }
                    out[n++] = (uint8_t)bit;
                    if (bit) {
                        out[n++] = neg[c];
                        sig[c] = 1;
                        rem_start = k + 1;
                        for (i = 0; i < nrem - rem_start; i++)
                            remaining[i] = remaining[rem_start + i];
                        nrem -= rem_start;
                        hit = 1;
                        break;
                    }
                }
                if (done || !hit) break;
            }
            if (done) break;
        }
    }
    return n;
}

/* Blocks of a (rows, cols) float32 array, edge-replicated (codec:157-164). */
static void gather_block(const float* a, int64_t rows, int64_t cols,
                         int64_t brow, int64_t bcol, float* blk) {
    for (int i = 0; i < 4; i++) {
        int64_t r = brow * 4 + i;
        if (r > rows - 1) r = rows - 1;
        for (int j = 0; j < 4; j++) {
            int64_t c = bcol * 4 + j;
            if (c > cols - 1) c = cols - 1;
            blk[4 * i + j] = a[r * cols + c];
        }
    }
}

/* codec:186-190 */
static uint16_t block_exponent(const float* blk) {
    float mx = 0.0f;
    for (int i = 0; i < 16; i++) {
        float a = fabsf(blk[i]);
        if (a > mx) mx = a;
    }
    if (!(mx > 0.0f)) return 0;
    int e;
    frexp((double)mx, &e);
    return (uint16_t)(e + ORC_EMAX_BIAS);
}

/* codec:193-198 + :137-142 + :239-243.  Returns 0, or -1 on overflow. */
static int block_coefficients(const float* blk, uint16_t code, int64_t* coef_seq) {
    int64_t t[16];
    int i;
    if (code == 0) {
        for (i = 0; i < 16; i++) coef_seq[i] = 0;
        return 0;
    }
    int emax = (int)code - ORC_EMAX_BIAS;
    double scale = ldexp(1.0, ORC_QUANT_BITS - emax);
    for (i = 0; i < 16; i++) t[i] = (int64_t)nearbyint((double)blk[i] * scale);
    for (i = 0; i < 4; i++)  /* rows */
        fwd_lift(&t[i * 4 + 0], &t[i * 4 + 1], &t[i * 4 + 2], &t[i * 4 + 3]);
    for (i = 0; i < 4; i++)  /* columns */
        fwd_lift(&t[0 * 4 + i], &t[1 * 4 + i], &t[2 * 4 + i], &t[3 * 4 + i]);
    for (i = 0; i < 16; i++) {
        coef_seq[i] = t[SEQUENCY[i]];
        int64_t a = coef_seq[i] < 0 ? -coef_seq[i] : coef_seq[i];
        if (a >= ((int64_t)1 << ORC_N_PLANES)) return -1;
    }
    return 0;
}

/* codec:271-293 for one block: smallest verified plane count, or 28 (raw). */
static int select_planes_one(const float* blk, const int valid[16], uint16_t code,
                             const uint32_t* mag, const uint8_t* neg, double tol) {
    for (int t = 0; t <= ORC_N_PLANES; t++) {
        unsigned shift = (unsigned)(ORC_N_PLANES - t);
        uint32_t tmag[16];
        float dec[16];
        for (int i = 0; i < 16; i++) tmag[i] = (uint32_t)(((uint64_t)mag[i] >> shift) << shift);
        reconstruct_one(tmag, neg, code, 0, NULL, dec);
        double emax = 0.0;
        int nan_seen = 0;
        for (int i = 0; i < 16; i++) {
            if (!valid[i]) continue;
            double e = fabs((double)dec[i] - (double)blk[i]);
            if (e != e) nan_seen = 1;
            if (e > emax) emax = e;
        }
        if (!nan_seen && emax <= tol) return t;
    }
    return ORC_N_PLANES + 1;
}

/* Full compress of one array.  mode 0 rate (param=bpv), 1 precision
 * (param=planes), 2 accuracy (tol).  Two calls: with payload == NULL it
 * returns total bits (and fills offsets); then call again with a
 * zeroed payload buffer of ceil(bits/8) bytes.  Returns -1 on coefficient
 * overflow (codec:240-241).                                              */
int64_t orc_compress(const float* a, int64_t rows, int64_t cols, int mode,
                     double param, uint64_t* offsets, uint8_t* payload) {
    int64_t br = (rows + 3) / 4, bc = (cols + 3) / 4, nb = br * bc;
    int budget = 0, has_raw = 0, planes_fixed = ORC_N_PLANES;
    if (mode == 0) budget = (int)param * 16;
    else if (mode == 1) planes_fixed = (int)param < ORC_N_PLANES ? (int)param : ORC_N_PLANES;
    else has_raw = 1;
    double tol = param;

    uint16_t* lens = (uint16_t*)malloc((size_t)nb * sizeof(uint16_t));
    if (!lens) return -2;
    int overflow = 0;
    int64_t b;
    /* pass 1: per-block length (identical encode, discarded bits) */
#pragma omp parallel
    {
        uint8_t* tmp = (uint8_t*)malloc(ORC_MAX_BLOCK_BITS + 64);
#pragma omp for schedule(static)
        for (b = 0; b < nb; b++) {
            float blk[16];
            int64_t coef[16], magl[16];
            uint32_t mag[16], rw[16];
            uint8_t neg[16];
            int valid[16];
            int64_t brow = b / bc, bcol = b % bc;
            gather_block(a, rows, cols, brow, bcol, blk);
            uint16_t code = block_exponent(blk);
            if (block_coefficients(blk, code, coef) < 0) {
#pragma omp atomic write
                overflow = 1;
                lens[b] = 0;
                continue;
            }
            for (int i = 0; i < 16; i++) {
                magl[i] = coef[i] < 0 ? -coef[i] : coef[i];
                mag[i] = (uint32_t)magl[i];
                neg[i] = coef[i] < 0;
            }
            int planes = planes_fixed, raw = 0;
            if (has_raw) {
                for (int i = 0; i < 4; i++)
                    for (int j = 0; j < 4; j++)
                        valid[4 * i + j] = (brow * 4 + i < rows) && (bcol * 4 + j < cols);
                planes = select_planes_one(blk, valid, code, mag, neg, tol);
                if (planes > ORC_N_PLANES) { raw = 1; planes = 0; }
                memcpy(rw, blk, sizeof(rw));
            }
            int n = encode_one(magl, neg, code, planes, raw, rw, ORC_N_PLANES,
                               budget, has_raw, tmp);
            if (budget) n = budget;
            lens[b] = (uint16_t)n;
        }
        free(tmp);
    }
    if (overflow) { free(lens); return -1; }
    uint64_t total = 0;
    for (b = 0; b < nb; b++) { offsets[b] = total; total += lens[b]; }
    if (payload) {
        /* pass 2: emit bits at their offsets.  Blocks share boundary bytes,
         * so write whole bytes from a per-thread range of blocks.          */
        int nth = orc_num_threads();
        int64_t chunk = (nb + nth - 1) / nth;
        int64_t t;
#pragma omp parallel for schedule(static, 1)
        for (t = 0; t < nth; t++) {
            uint8_t* tmp = (uint8_t*)calloc(ORC_MAX_BLOCK_BITS + 64, 1);
            int64_t b0 = t * chunk, b1 = b0 + chunk < nb ? b0 + chunk : nb;
            /* boundary bytes between chunks are OR-ed atomically */
            for (int64_t bb = b0; bb < b1; bb++) {
                float blk[16];
                int64_t coef[16], magl[16];
                uint32_t mag[16], rw[16];
                uint8_t neg[16];
                int valid[16];
                int64_t brow = bb / bc, bcol = bb % bc;
                gather_block(a, rows, cols, brow, bcol, blk);
                uint16_t code = block_exponent(blk);
                block_coefficients(blk, code, coef);
                for (int i = 0; i < 16; i++) {
                    magl[i] = coef[i] < 0 ? -coef[i] : coef[i];
                    mag[i] = (uint32_t)magl[i];
                    neg[i] = coef[i] < 0;
                }
                int planes = planes_fixed, raw = 0;
                if (has_raw) {
                    for (int i = 0; i < 4; i++)
                        for (int j = 0; j < 4; j++)
                            valid[4 * i + j] = (brow * 4 + i < rows) && (bcol * 4 + j < cols);
                    planes = select_planes_one(blk, valid, code, mag, neg, tol);
                    if (planes > ORC_N_PLANES) { raw = 1; planes = 0; }
                    memcpy(rw, blk, sizeof(rw));
                }
                memset(tmp, 0, ORC_MAX_BLOCK_BITS + 64);
                int n = encode_one(magl, neg, code, planes, raw, rw, ORC_N_PLANES,
                                   budget, has_raw, tmp);
                if (budget) n = budget; /* zero padded (tmp cleared) */
                uint64_t pos = offsets[bb];
                for (int i = 0; i < n; i++, pos++) {
                    if (tmp[i]) {
                        uint8_t m = (uint8_t)(0x80u >> (pos & 7));
#pragma omp atomic update
                        payload[pos >> 3] |= m;
                    }
                }
            }
            free(tmp);
        }
    }
    free(lens);
    return (int64_t)total;
}

/* ------------------------------------------------------------------------ */
/* thermal: thermal:98-109 (thermal_step), :112-117 (thermal_interpolate).  */
/* scipy csr_matvec: y[i] = sum_j data[j]*x[col[j]] in CSR order, fp64.     */
/* ------------------------------------------------------------------------ */
void orc_thermal_step(const int64_t* indptr, const int32_t* indices,
                      const double* data, int64_t n, const float* B,
                      const float* T_k, const float* u_k, float* T_next) {
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; i++) {
        double acc = 0.0;
        for (int64_t jj = indptr[i]; jj < indptr[i + 1]; jj++)
            acc += data[jj] * (double)T_k[indices[jj]];
        acc += (double)B[i] * (double)u_k[i];
        T_next[i] = (float)acc;
    }
}

void orc_csr_matvec_f32out(const int64_t* indptr, const int32_t* indices,
                           const double* data, int64_t n, const float* x,
                           float* y) {
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; i++) {
        double acc = 0.0;
        for (int64_t jj = indptr[i]; jj < indptr[i + 1]; jj++)
            acc += data[jj] * (double)x[indices[jj]];
        y[i] = (float)acc;
    }
}

/* K:228-283 encode_blocks from per-block arrays.  Two calls: payload NULL
 * returns total bits and fills offsets; then emit into a zeroed payload.   */
int64_t orc_encode_blocks(const uint32_t* mag, const uint8_t* neg, const uint16_t* emax,
                          const uint8_t* planes, const uint8_t* raw_mask,
                          const uint32_t* raw_words, int64_t nb, int budget,
                          int has_raw_flag, uint64_t* offsets, uint8_t* payload) {
    uint8_t* tmp = (uint8_t*)calloc(ORC_MAX_BLOCK_BITS + (budget > 0 ? budget : 0) + 64, 1);
    uint64_t total = 0;
    for (int64_t b = 0; b < nb; b++) {
        int64_t magl[16];
        for (int i = 0; i < 16; i++) magl[i] = mag[16 * b + i];
        offsets[b] = total;
        memset(tmp, 0, ORC_MAX_BLOCK_BITS + (budget > 0 ? budget : 0) + 64);
        int n = encode_one(magl, neg + 16 * b, emax[b], planes[b],
                           has_raw_flag ? raw_mask[b] : 0, raw_words + 16 * b,
                           ORC_N_PLANES, budget, has_raw_flag, tmp);
        if (budget) n = budget;
        if (payload)
            for (int i = 0; i < n; i++)
                if (tmp[i]) payload[(total + i) >> 3] |= (uint8_t)(0x80u >> ((total + i) & 7));
        total += n;
    }
    free(tmp);
    return (int64_t)total;
}
