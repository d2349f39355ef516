"""Adversarial LLR stream for the 16-bit metric range of the 16x2 kernels.

Greedy search over max-magnitude LLR tuples that maximises the path-metric
spread after each stage (2-step lookahead, random tie-breaks).  The 16x2
kernels' range argument needs spread <= 256 * W (W = the code's maximum
output-difference weight over K-1 stages: 11 for (171,133), 15 for the r1/3
(133,171,165), 13 for K=9 (753,561)).  (171,133) reaches 2048 of 2816.
usage: python make_adversarial.py [k7r2|k7r3|k9r2]
Output: tests/golden/adversarial_<code>.npz (int8 (N, B)).
"""
import itertools, numpy as np, sys
CODES={"k7r2": (7, (0o171,0o133)), "k7r3": (7, (0o133,0o171,0o165)), "k9r2": (9, (0o753,0o561))}
name=sys.argv[1] if len(sys.argv)>1 else "k7r2"
K, G = CODES[name]; S=1<<(K-1)
def parity(x): return bin(x).count("1")&1
pred0=np.array([(2*(j%(S//2))) for j in range(S)]); pred1=pred0+1
def pat(i,u): reg=(u<<(K-1))|i; return [1-2*parity(g&reg) for g in G]
sg0=np.array([pat(pred0[j], j>>(K-2)) for j in range(S)]); sg1=np.array([pat(pred1[j], j>>(K-2)) for j in range(S)])
if name=="k7r2":
    cands=[np.array(c) for c in [(127,127),(127,-128),(-128,127),(-128,-128),(0,0),(127,0),(0,127),(-128,0),(0,-128)]]
else:  # max-magnitude corners first (the 2-step lookahead scans cands[:4])
    corners=[np.array(c) for c in itertools.product((127,-128), repeat=len(G))]
    cands=corners+[np.array(c) for c in itertools.product((127,-128,0), repeat=len(G)) if 0 in c]
trials=40 if name=="k7r2" else 20
def step(M,l):
    return np.maximum(M[pred0]+sg0@l, M[pred1]+sg1@l)
rng=np.random.default_rng(0)
best_overall=0; seqs=[]
for trial in range(trials):
    M=np.zeros(S,np.int64); seq=[]
    for t in range(600):
        # greedy with random tie-break + 2-step lookahead on a random subset
        scores=[]
        for c in cands:
            M1=step(M,c)
            sp=max(M1.max()-M1.min(), max((step(M1,c2).max()-step(M1,c2).min()) for c2 in cands[:4]))
            scores.append(sp + rng.random()*0.5)
        c=cands[int(np.argmax(scores))] if rng.random()>0.1 else cands[rng.integers(len(cands))]
        M=step(M,c); M-=M.max(); seq.append(c)
        best_overall=max(best_overall, -M.min())
    seqs.append(np.array(seq))
W={"k7r2":11,"k7r3":15,"k9r2":13}[name]
print("max spread observed", best_overall, "bound", 256*W)
import os
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), f"adversarial_{name}.npz"), llr=np.concatenate(seqs).astype(np.int8), max_spread=np.int64(best_overall))
