"""Survivor-history live set of the 16x2 decoder in L2.

Model: every CTA slot decodes tiles back to back; tile t's stored history groups
gs = 0..nbs-1 are written at group end gs + (b_lo - skip) of tile t and read by
tile t's traceback during tile t+1 (`k` groups per group end: the shipped kernel
walks k = 1; `k` = inf is an instant traceback at the tile end).  A group slice
is (CTAs x threads x bytes per thread); its L2 occupancy is slice x lifetime /
tile period.  Whatever is live beyond the L2 capacity thrashes (a cyclic reuse
pattern larger than an LRU-like cache misses almost always).

    python tools/live_set_model.py            # config 2 (F=256, V=42), 2 CTAs/SM
    python tools/live_set_model.py --ctas 1   # one CTA per SM
"""
import argparse


def live_set(nbs=100, b_lo=20, skip_groups=6, ng=120, k=1.0, ctas=296, threads=128, bytes_per_group=64,
             onchip_groups=0):
    period = ng - skip_groups  # group ends per tile
    total = 0.0
    for gs in range(onchip_groups, nbs):
        write = gs + b_lo - skip_groups
        read = period + (nbs - 1 - gs) / k
        total += read - write
    return total * ctas * threads * bytes_per_group / period


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctas", type=int, default=2, help="CTAs per SM")
    ap.add_argument("--sms", type=int, default=148)
    a = ap.parse_args()
    ctas = a.ctas * a.sms
    slot = ctas * 128 * 64 * 100 / 1e6
    print(f"slot (1 tile of histories per CTA): {slot:.0f} MB at {ctas} CTAs")
    for k in (1, 2, 4, float("inf")):
        for bpg, tag in ((64, "3-bit fields, 4 states/word (shipped)"), (48, "dense 1 bit/state/stage")):
            mb = live_set(k=k, ctas=ctas, bytes_per_group=bpg) / 1e6
            print(f"traceback {k:>3} groups/group end, {tag:40s}: live {mb:6.0f} MB  (L2 126 MB)")


if __name__ == "__main__":
    main()
