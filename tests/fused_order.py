"""CPU model of the fused kernel's summation order (test infrastructure).

`k_decode_gemv` with the exact evaluation (csrc/whff_b200.cu) computes each
row of a 4-row block-row as follows; this module restates it with numpy's
IEEE binary32/binary64 arithmetic, so tests can require the device result
bit for bit rather than within the reference's bound:

* block column b = 32 g + l belongs to lane l of group g; group g belongs to
  virtual warp g mod 32;
* lane l of virtual warp w starts at +0.0 and, for its groups g = w, w + 32,
  ... in order, adds for each column j = 0..3 of the block the product
  x[i, 4b + j] * v[4b + j] (binary32 product; policy "mixed": rounded to
  binary32 then added in binary64; "double": binary64 product and sum;
  "single": binary32 sum); padded columns add x = 0, v = 0;
* the 32 lane partials of a virtual warp are combined by the xor butterfly
  a[l] <- a[l] + a[l ^ o], o = 16, 8, 4, 2, 1, and the 32 virtual-warp sums
  by the same butterfly; the row is binary32(sum) ("mixed"/"double") or the
  binary32 sum ("single").

The decoded matrix must be the codec's bit-exact words (oracle decompress).
`fused_coefficient` models the coefficient-domain evaluation the same way
(binary32 FMAs emulated exactly, with a rational fallback for the rare
binary64 results that land on a binary32 tie).
"""

import numpy as np

KVW = 32


def _butterfly(a, offsets=(16, 8, 4, 2, 1)):
    """a: (..., 32) -> the xor-butterfly sum (identical in every lane), lane 0."""
    idx = np.arange(32)
    for o in offsets:
        a = a + a[..., idx ^ o]
    return a[..., 0]


def fused_exact(words, v, policy="mixed"):
    """Rows of C @ v in the fused kernel's order; words (rows, cols) binary32."""
    words = np.asarray(words, dtype=np.float32)
    v = np.asarray(v, dtype=np.float32)
    rows, cols = words.shape
    bc = (cols + 3) // 4
    gpr = (bc + 31) // 32
    br = (rows + 3) // 4
    X = np.zeros((br * 4, gpr * 128), np.float32)
    X[:rows, :cols] = words
    V = np.zeros(gpr * 128, np.float32)
    V[:cols] = v
    # [block-row, row i, group g, lane l, column j]
    X = X.reshape(br, 4, gpr, 32, 4)
    V = V.reshape(gpr, 32, 4)
    if policy == "single":
        acc_t = np.float32
        P = (X * V).astype(np.float32)
    elif policy == "mixed":
        acc_t = np.float64
        P = (X * V).astype(np.float32).astype(np.float64)
    else:
        acc_t = np.float64
        P = X.astype(np.float64) * V.astype(np.float64)
    # lane partials per virtual warp: acc[br, i, vw, l]
    acc = np.zeros((br, 4, KVW, 32), acc_t)
    nk = (gpr + KVW - 1) // KVW
    for k in range(nk):
        for vw in range(KVW):
            g = vw + KVW * k
            if g >= gpr:
                continue
            for j in range(4):
                acc[:, :, vw, :] = acc[:, :, vw, :] + P[:, :, g, :, j]
    per_vw = _butterfly(acc)                 # (br, 4, KVW)
    tot = _butterfly(per_vw)                 # (br, 4)
    out = tot.astype(np.float32).reshape(br * 4)[:rows]
    return out


# ---------------------------------------------------------------------------
# coefficient-domain evaluation (EVAL_COEFF)
# ---------------------------------------------------------------------------
# G = the real-valued inverse lift (csrc/whff_b200.cu c_G); SEQ = raster
# position of the i-th coefficient in sequency order (codec.py:40).
G = np.array([[1.0, 1.5, -1.0, -0.25],
              [1.0, 0.5, 1.0, 1.25],
              [1.0, -0.5, 1.0, -1.25],
              [1.0, -1.5, -1.0, 0.25]], np.float32)
SEQ = [0, 1, 4, 2, 5, 8, 3, 6, 9, 12, 7, 10, 13, 11, 14, 15]
EMAX_BIAS, QUANT_BITS = 160, 26


def _round_f32(x):
    """Correctly rounded binary32 of a Fraction (ties to even)."""
    from fractions import Fraction
    c = np.float32(float(x))
    best = None
    for cand in (np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))):
        err = abs(Fraction(float(cand)) - x)
        key = (err, int(cand.view(np.uint32)) & 1)
        if best is None or key < best[0]:
            best = (key, cand)
    return best[1]


def fma32(a, b, c):
    """Elementwise binary32 fma(a, b, c), exactly rounded."""
    from fractions import Fraction
    a, b, c = np.broadcast_arrays(*(np.atleast_1d(np.asarray(t, np.float32)) for t in (a, b, c)))
    r = a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)   # a*b exact
    out = r.astype(np.float32)
    f = out.astype(np.float64)
    toward = np.where(r > f, np.float32(np.inf), np.float32(-np.inf)).astype(np.float32)
    mid = (f + np.nextafter(out, toward).astype(np.float64)) / 2
    amb = (r == mid) & (r != f)            # binary64 rounding landed on a binary32 tie
    for idx in zip(*np.nonzero(amb)):
        out[idx] = _round_f32(Fraction(float(a[idx])) * Fraction(float(b[idx]))
                              + Fraction(float(c[idx])))
    return out


def fma64(a, b, c):
    """Scalar binary64 fma, exactly rounded."""
    from fractions import Fraction
    return float(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def fused_coefficient(orc, stream, v, policy="mixed"):
    """Rows of the coefficient-domain evaluation in the fused kernel's order,
    from the oracle's decode_blocks fields of a host stream."""
    v = np.asarray(v, np.float32)
    rows, cols = stream.rows, stream.cols
    code, _ = orc.mode_kind(stream.mode)
    payload = np.ascontiguousarray(stream.payload, np.uint8)
    index = np.ascontiguousarray(stream.block_index, np.uint64)
    seg = orc.segment_lengths(stream.mode, payload.size, index)
    mag, neg, emax, raw, raw_words, _ = orc.decode_blocks(
        payload, index, seg, 27, orc.planes_limit_for(stream.mode), code == 2)
    words = orc.decompress(stream)
    bc = (cols + 3) // 4
    br = (rows + 3) // 4
    gpr = (bc + 31) // 32
    nbp = gpr * 32
    # per block-column u = G^T v (binary64 sum, binary32 result; k_coeff_prep)
    vp = np.zeros(nbp * 4, np.float32)
    vp[:cols] = v
    V = vp.reshape(nbp, 4)
    U = np.zeros((nbp, 4), np.float32)
    for k in range(4):
        t = np.zeros(nbp, np.float64)
        for j in range(4):
            t = t + np.float64(G[j, k]) * V[:, j].astype(np.float64)
        U[:, k] = t.astype(np.float32)
    # per-block fields, padded to (br, nbp)
    def pad(a, fill=0):
        out = np.full((br, nbp) + a.shape[1:], fill, a.dtype)
        out[:, :bc] = a.reshape((br, bc) + a.shape[1:])
        return out
    mag, neg, emax, raw = pad(mag), pad(neg), pad(emax), pad(raw)
    k = emax.astype(np.int64) - EMAX_BIAS - QUANT_BITS
    ok = (raw == 0) & ((emax == 0) | ((k >= -126) & (k <= 100)))
    use = ok & (emax != 0)
    # sink: w[a] = fma(q, u[j], w[a]) over significant coefficients in order
    w = np.zeros((br, nbp, 4), np.float32)
    for c in range(16):
        pos = SEQ[c]
        a, j = pos >> 2, pos & 3
        q = mag[:, :, c].astype(np.float32)
        q = np.where(neg[:, :, c] != 0, -q, q).astype(np.float32)
        sig = mag[:, :, c] != 0
        nw = fma32(q, np.broadcast_to(U[None, :, j], q.shape), w[:, :, a])
        w[:, :, a] = np.where(sig, nw, w[:, :, a])
    sc = np.zeros((br, nbp), np.float32)
    kk = np.clip(k, -126, 100)
    sc[:] = np.ldexp(np.float32(1.0), kk).astype(np.float32)
    T = (w * sc[:, :, None]).astype(np.float32)               # exact scaling (or underflow RN)
    # fallback blocks: exact spatial products (raw escapes, extreme scales)
    fb = ~ok & ((raw != 0) | (emax != 0))
    Xp = np.zeros((br * 4, nbp * 4), np.float32)
    Xp[:rows, :cols] = words
    X = Xp.reshape(br, 4, nbp, 4).transpose(0, 2, 1, 3)       # [br, bcol, i, j]
    single = policy == "single"
    acc_t = np.float32 if single else np.float64
    Pf = (X * V[None, :, None, :]).astype(np.float32)          # binary32 products
    # lane accumulation: vw over groups, blocks = 32 lanes of a group
    D = np.zeros((br, 32, 32, 4), acc_t)                       # [br, vw, lane, a]
    R = np.zeros((br, 32, 32, 4), acc_t)                       # [br, vw, lane, i]
    nk = (gpr + 31) // 32
    for kq in range(nk):
        for vw in range(32):
            g = vw + 32 * kq
            if g >= gpr:
                continue
            sl = slice(32 * g, 32 * g + 32)
            t = T[:, sl, :].astype(acc_t)
            D[:, vw] = np.where(use[:, sl, None], D[:, vw] + t, D[:, vw])
            m = fb[:, sl]
            for i in range(4):
                r = R[:, vw, :, i]
                for jj in range(4):
                    r = np.where(m, r + Pf[:, sl, i, jj].astype(acc_t), r)
                R[:, vw, :, i] = r
    Dv = _butterfly(np.moveaxis(D, 2, -1))                     # [br, vw, a]
    Rv = _butterfly(np.moveaxis(R, 2, -1))                     # [br, vw, i]
    Dt = _butterfly(np.moveaxis(Dv, 1, -1))                    # [br, a]
    Rt = _butterfly(np.moveaxis(Rv, 1, -1))                    # [br, i]
    out = np.zeros(br * 4, np.float32)
    for b in range(br):
        for i in range(4):
            if single:
                t = np.float32(Rt[b, i])
                for a in range(4):
                    t = fma32(G[i, a], Dt[b, a], t)[0]
                out[4 * b + i] = t
            else:
                t = float(Rt[b, i])
                for a in range(4):
                    t = fma64(G[i, a], Dt[b, a], t)
                out[4 * b + i] = np.float32(t)
    return out[:rows]


# ---------------------------------------------------------------------------
# tile-packed layout (k_pk_gemv, csrc/whff_packed.cu)
# ---------------------------------------------------------------------------
# * bands of 4 block-rows; a band's segments (SEG_TILES tiles of 32
#   block-columns, per stream mode: packed_host.seg_tiles_for) are dealt to
#   32 virtual warps (segment s -> virtual warp
#   s mod 32); lane l of tile t of segment s = column 32 (SEG_TILES s + t) + l;
# * lane accumulators per (band row i, row r) add, per block, the
#   coefficient-domain term binary32(w_r * 2^k) (w as fused_coefficient,
#   every coefficient applied, q exact or rounded for |q| >= 2^24) or the
#   exact products x[r, j] * v[j] in column order;
# * exceptions (raw escapes, scales outside 2^-126..2^100) are left out of
#   the lane sums; per segment, in (tile, row, lane) order, the warp adds
#   (p0 + p1) + (p2 + p3) of each of their rows to a per-warp sum R;
# * lane butterfly, virtual-warp butterfly; y = binary32(R + sum_a G D_a) in
#   the coefficient domain (fma order a = 0..3 onto R), binary32(D + R)
#   exactly.

def _exceptions(emax, raw):
    k = emax.astype(np.int64) - EMAX_BIAS - QUANT_BITS
    return (raw != 0) | ((emax != 0) & ~((k >= -126) & (k <= 100)))


def packed_model(orc, stream, v, policy="mixed", evaluation="coefficient"):
    v = np.asarray(v, np.float32)
    rows, cols = stream.rows, stream.cols
    code, _ = orc.mode_kind(stream.mode)
    payload = np.ascontiguousarray(stream.payload, np.uint8)
    index = np.ascontiguousarray(stream.block_index, np.uint64)
    seg = orc.segment_lengths(stream.mode, payload.size, index)
    mag, neg, emax, raw, raw_words, _ = orc.decode_blocks(
        payload, index, seg, 27, orc.planes_limit_for(stream.mode), code == 2)
    words = orc.decompress(stream)
    bc, br = (cols + 3) // 4, (rows + 3) // 4
    nband = (br + 3) // 4
    ntile = (bc + 31) // 32
    from packed_host import seg_tiles_for
    SEG_TILES = seg_tiles_for(stream.mode)
    nsegb = (ntile + SEG_TILES - 1) // SEG_TILES
    nbp = nsegb * SEG_TILES * 32
    single = policy == "single"
    acc_t = np.float32 if single else np.float64
    vp = np.zeros(nbp * 4, np.float32)
    vp[:cols] = v
    V = vp.reshape(nbp, 4)
    exc = np.zeros((nband * 4, nbp), bool)
    exc[:br, :bc] = _exceptions(emax, raw).reshape(br, bc)
    Xp = np.zeros((nband * 16, nbp * 4), np.float32)
    Xp[:rows, :cols] = words
    X = Xp.reshape(nband * 4, 4, nbp, 4).transpose(0, 2, 1, 3)      # [brow, bcol, r, j]
    Pf = (X * V[None, :, None, :]).astype(np.float32)
    if policy == "double":
        Pf = X.astype(np.float64) * V[None, :, None, :].astype(np.float64)
    Pa = Pf.astype(acc_t)
    if evaluation == "coefficient":
        U = np.zeros((nbp, 4), np.float32)
        for kk in range(4):
            t = np.zeros(nbp, np.float64)
            for j in range(4):
                t = t + np.float64(G[j, kk]) * V[:, j].astype(np.float64)
            U[:, kk] = t.astype(np.float32)
        def pad(a):
            out = np.zeros((nband * 4, nbp) + a.shape[1:], a.dtype)
            out[:br, :bc] = a.reshape((br, bc) + a.shape[1:])
            return out
        M, N, E = pad(mag), pad(neg), pad(emax)
        w = np.zeros((nband * 4, nbp, 4), np.float32)
        for c in range(16):
            pos = SEQ[c]
            a, j = pos >> 2, pos & 3
            q = M[:, :, c].astype(np.float32)            # rounded to binary32 above 2^24
            q = np.where(N[:, :, c] != 0, -q, q).astype(np.float32)
            if c == 0:
                w[:, :, 0] = (q * U[None, :, 0]).astype(np.float32)
            else:
                w[:, :, a] = fma32(q, np.broadcast_to(U[None, :, j], q.shape), w[:, :, a])
        kk = np.clip(E.astype(np.int64) - EMAX_BIAS - QUANT_BITS, -126, 100)
        sc = np.ldexp(np.float32(1.0), kk).astype(np.float32)
        use = (E != 0) & ~exc
        T = np.where(use[:, :, None], (w * sc[:, :, None]).astype(np.float32), np.float32(0))
        T = T.astype(acc_t)
    out = np.zeros(nband * 16, np.float32)
    for band in range(nband):
        R = np.zeros((32, 16), acc_t)                 # [vw, 4 i + r]
        # k_pk_gemv2's order, both evaluations: per segment, per-lane sums over
        # the segment's tiles -- coefficient: binary32 (one FMA rounding per
        # term), reduced over the warp in binary32 (xor 16, 8, 4, 2, 1) and
        # converted once; exact: the policy's accumulator (binary64 for
        # mixed), reduced over the warp in it -- accumulated per segment in
        # the virtual warp's order
        Dv_acc = np.zeros((32, 16), acc_t)
        for vw in range(32):
            for sb in range(vw, nsegb, 32):
                Sg = np.zeros((32, 4, 4), np.float32)          # [lane, i, r] (coefficient)
                Se = np.zeros((32, 4, 4), acc_t)               # [lane, i, r] (exact)
                for tt in range(SEG_TILES):
                    cs = (SEG_TILES * sb + tt) * 32 + np.arange(32)
                    for i in range(4):
                        b = 4 * band + i
                        if evaluation == "coefficient":
                            Sg[:, i, :] = (Sg[:, i, :] + T[b, cs, :].astype(np.float32)).astype(np.float32)
                        else:
                            m = ~exc[b, cs]
                            for r in range(4):
                                for j in range(4):
                                    Se[:, i, r] = np.where(m, Se[:, i, r] + Pa[b, cs, r, j], Se[:, i, r])
                if evaluation == "coefficient":
                    # seg_reduce: the whole butterfly in binary32, then one
                    # conversion to the accumulator
                    Dseg = Sg.reshape(32, 16)                          # [lane, m = 4 i + r]
                    Dv_acc[vw] = Dv_acc[vw] + _butterfly(np.moveaxis(Dseg, 0, -1)).astype(acc_t)
                else:
                    Dv_acc[vw] = Dv_acc[vw] + _butterfly(np.moveaxis(Se.reshape(32, 16), 0, -1))
                for tt in range(SEG_TILES):
                    for i in range(4):
                        b = 4 * band + i
                        for lane in range(32):
                            col = (SEG_TILES * sb + tt) * 32 + lane
                            if col >= bc or b >= br or not exc[b, col]:
                                continue
                            for r in range(4):
                                p = Pa[b, col, r]
                                R[vw, 4 * i + r] = R[vw, 4 * i + r] + ((p[0] + p[1]) + (p[2] + p[3]))
        Dv = Dv_acc.reshape(32, 4, 4)
        Dt = _butterfly(np.moveaxis(Dv, 0, -1))        # [i, r]
        Rt = _butterfly(np.moveaxis(R, 0, -1))         # [16]
        for i in range(4):
            for r in range(4):
                if evaluation == "coefficient":
                    if single:
                        t = np.float32(Rt[4 * i + r])
                        for a in range(4):
                            t = fma32(G[r, a], Dt[i, a], t)[0]
                        out[16 * band + 4 * i + r] = t
                    else:
                        t = float(Rt[4 * i + r])
                        for a in range(4):
                            t = fma64(G[r, a], Dt[i, a], t)
                        out[16 * band + 4 * i + r] = np.float32(t)
                else:
                    if single:
                        out[16 * band + 4 * i + r] = np.float32(Dt[i, r]) + np.float32(Rt[4 * i + r])
                    else:
                        out[16 * band + 4 * i + r] = np.float32(float(Dt[i, r]) + float(Rt[4 * i + r]))
    return out[:rows]
