"""numpy model of csrc/vt_tiles.cu driven by the SAME host tables
(paper_2011_13579_b200.tiles): each tile op D = A x B + C in float32 (exact here),
rounded to binary16 for accumulator="half", the later candidate winning ties,
matrix._traceback_steps.  Checked on the CPU against decode_matrix_batch results
the reference produced (tests/golden/golden_r2.npz, kind "tile")."""
import numpy as np

from paper_2011_13579_b200.tiles import fragment_tables, radix2_tiles, radix4_tiles


def _dense(tab, t):
    """Rebuild tile t's A and the B / C gather maps from the per-lane fragment tables
    (so the model exercises the fragment layout the kernel uses)."""
    a = np.zeros((16, 16), dtype=np.float32)
    bsel = np.full((16, 16), -1, dtype=np.int64)
    cst = np.full((16, 16), -1, dtype=np.int64)
    for lane in range(32):
        g, q = lane >> 2, lane & 3
        for r, (row, col) in enumerate(((g, 2 * q), (g + 8, 2 * q), (g, 2 * q + 8), (g + 8, 2 * q + 8))):
            w = int(tab["a_frag"][t, lane, r])
            a[row, col] = np.array(w & 0xFFFF, dtype=np.uint16).view(np.float16)
            a[row, col + 1] = np.array(w >> 16, dtype=np.uint16).view(np.float16)
        for nb in range(2):
            for i, row in enumerate((2 * q, 2 * q + 1, 2 * q + 8, 2 * q + 9)):
                bsel[row, nb * 8 + g] = tab["b_sel"][t, lane, nb * 4 + i]
            c0 = nb * 8 + 2 * q
            for i, (row, col) in enumerate(((g, c0), (g, c0 + 1), (g + 8, c0), (g + 8, c0 + 1))):
                cst[row, col] = tab["c_state"][t, lane, nb * 4 + i]
    return a, bsel, cst


def decode(llr_fbn, spec, radix, optimized, half, renormalize):
    f, b, n = llr_fbn.shape
    s = spec.num_states
    progs = {2: fragment_tables(radix2_tiles(spec))}
    if radix == 4:
        progs[4] = fragment_tables(radix4_tiles(spec, optimized))
    dense = {r: [_dense(p, t) for t in range(p["ntiles"])] for r, p in progs.items()}
    lam = np.zeros((f, s), dtype=np.float32)
    off = np.zeros(f)
    steps = []
    t = 0
    mmas = 0
    while t < n:
        r = 4 if (radix == 4 and t + 1 < n) else 2
        p = progs[r]
        llr = llr_fbn[:, :, t].astype(np.float32) if r == 2 else \
            np.concatenate([llr_fbn[:, :, t], llr_fbn[:, :, t + 1]], axis=1).astype(np.float32)
        new = np.zeros_like(lam)
        surv = np.zeros((f, s), dtype=np.uint8)
        for ti, (a, bsel, cst) in enumerate(dense[r]):
            bm = np.where(bsel >= 0, llr[:, np.maximum(bsel, 0)], 0.0).astype(np.float32)
            cm = np.where(cst >= 0, lam[:, np.maximum(cst, 0)], 0.0).astype(np.float32)
            with np.errstate(all="ignore"):
                d = (np.einsum("rk,fkc->frc", a, bm) + cm).astype(np.float32)
                if half:
                    d = d.astype(np.float16).astype(np.float32)
            mmas += 2
            flat = d.reshape(f, 256)
            for o in range(p["nout"]):
                st = p["out_state"][ti, o]
                if st < 0:
                    continue
                cand = flat[:, p["cand"][ti, o, :p["ncand"]]]
                k = p["ncand"] - 1 - np.argmax(cand[:, ::-1] >= cand.max(axis=1, keepdims=True), axis=1)
                new[:, st] = cand[np.arange(f), k]
                surv[:, st] = p["code"][ti, o][k]
        if renormalize:
            top = new.max(axis=1)
            off += top.astype(np.float64)
            with np.errstate(all="ignore"):
                new = new - top[:, None]
                if half:
                    new = new.astype(np.float16).astype(np.float32)
        lam = new
        steps.append((r, t, surv))
        t += 2 if r == 4 else 1
    final = lam.max(axis=1).astype(np.float64) + off
    k = spec.constraint_length
    j = np.argmax(lam, axis=1)
    bits = np.zeros((f, n), dtype=np.uint8)
    rows = np.arange(f)
    for r, t, sv in reversed(steps):
        if r == 2:
            bits[:, t] = j >> (k - 2)
            j = 2 * (j & (s // 2 - 1)) + sv[rows, j]
        else:
            y = j >> (k - 3)
            bits[:, t + 1] = y >> 1
            bits[:, t] = y & 1
            j = 4 * (j & ((1 << (k - 3)) - 1)) + sv[rows, j]
    return bits, final, mmas // 2
