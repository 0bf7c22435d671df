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
"""

import numpy as np

KVW = 32


def _butterfly(a):
    """a: (..., 32) -> the xor-butterfly sum (identical in every lane), lane 0."""
    idx = np.arange(32)
    for o in (16, 8, 4, 2, 1):
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
