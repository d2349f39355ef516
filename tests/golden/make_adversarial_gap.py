"""Adversarial LLR streams for the subset-minimum renormalisation of the 16x2 kernels
(gen_kernels16.renorm_set): the kernels renormalise by R = min over a small state set T
instead of the exact minimum, which is safe while min_T Lambda - min Lambda <= 256 * W_T
(W_T from the weight table) and the span max Lambda - R stays <= Delta.

Greedy search over max-magnitude LLR tuples (random tie-breaks, 2-step lookahead) that
maximises the gap min_T Lambda - min Lambda for the generator's own sets T (both group
positions of the K=9 body), with the spread as a secondary score.
usage: python make_adversarial_gap.py [k7r3|k9r2|k7r2alt]
Output: tests/golden/adversarial_gap_<code>.npz (int8 (N, B), plus the largest gap seen).
"""
import itertools
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "paper_2011_13579_b200", "csrc"))
from gen_kernels16 import Gen16  # noqa: E402
from gen_kernels16m import Gen16M  # noqa: E402

CODES = {"k7r3": (7, (0o133, 0o171, 0o165)), "k9r2": (9, (0o753, 0o561)), "k7r2alt": (7, (0o171, 0o133))}
name = sys.argv[1] if len(sys.argv) > 1 else "k7r3"
K, G = CODES[name]
S = 1 << (K - 1)
if K == 9:
    g = Gen16M(name, K, G, 4)
    sets = [np.array(r[0]) for r in g.rsets]
elif name.endswith("alt"):  # the alternating form's renormalisation set (VT_ALT16)
    os.environ["VT_ALT16"] = "1"
    g = Gen16(name, K, G)
    sets = [np.array(g.alt_T)]
    g.Sb = g.Sb_alt
else:
    g = Gen16(name, K, G)
    sets = [np.array(g.rset)]


def parity(x):
    return bin(x).count("1") & 1


pred0 = np.array([2 * (j % (S // 2)) for j in range(S)])
pred1 = pred0 + 1


def pat(i, u):
    reg = (u << (K - 1)) | i
    return [1 - 2 * parity(gg & reg) for gg in G]


sg0 = np.array([pat(pred0[j], j >> (K - 2)) for j in range(S)])
sg1 = np.array([pat(pred1[j], j >> (K - 2)) for j in range(S)])
cands = [np.array(c) for c in itertools.product((127, -128), repeat=len(G))]
cands += [np.array(c) for c in itertools.product((127, -128, 0), repeat=len(G)) if 0 in c]


def step(M, ll):
    return np.maximum(M[pred0] + sg0 @ ll, M[pred1] + sg1 @ ll)


def gap(M):
    return max(int(M[T].min() - M.min()) for T in sets)


rng = np.random.default_rng(1)
best = 0
seqs = []
for trial in range(12):
    M = np.zeros(S, np.int64)
    seq = []
    for t in range(500):
        scores = []
        for c in cands:
            M1 = step(M, c)
            look = max(gap(step(M1, c2)) for c2 in cands[:2 ** len(G)])  # 2-step lookahead
            scores.append(max(gap(M1), look) + 0.01 * (M1.max() - M1.min()) + rng.random() * 0.5)
        c = cands[int(np.argmax(scores))] if rng.random() > 0.1 else cands[rng.integers(len(cands))]
        M = step(M, c)
        M -= M.min()
        seq.append(c)
        best = max(best, gap(M))
    seqs.append(np.array(seq))
print("max gap observed", best, "bound", g.Sb)
np.savez_compressed(os.path.join(HERE, f"adversarial_gap_{name}.npz"),
                    llr=np.concatenate(seqs).astype(np.int8), max_gap=np.int64(best))
