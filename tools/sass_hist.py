"""Summarise an ncu source page (--page source --csv --print-source sass):
executed warp instructions and stall samples per opcode, and per region.
usage: python tools/sass_hist.py src.csv [--regions]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
ops = collections.Counter(); st = collections.Counter()
tot = 0; tots = 0
seq = []
for r in data:
    try:
        n = int(r[ix["Instructions Executed"]]); s = int(r[ix["Warp Stall Sampling (All Samples)"]])
    except Exception:
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.rstrip(";")
    ops[op] += n; st[op] += s; tot += n; tots += s
    seq.append((r[ix["Address"]], src, n, s))
print(f"total warp instr {tot:,}  stall samples {tots:,}")
for op, n in ops.most_common(45):
    print(f"{op:28s} {n:14,d} {100*n/tot:6.2f}%  samples {100*st[op]/max(tots,1):6.2f}%")
if "--regions" in sys.argv:
    # contiguous runs of equal execution count = basic blocks
    cur = None; start = None; cnt = 0; smp = 0; ninst = 0
    out = []
    for a, src, n, s in seq:
        if n != cur:
            if cur is not None: out.append((start, ninst, cur, smp))
            cur = n; start = a; ninst = 0; smp = 0
        ninst += 1; smp += s
    out.append((start, ninst, cur, smp))
    for start, ninst, n, smp in sorted(out, key=lambda x: -x[1] * x[2])[:30]:
        print(f"{start} len {ninst:5d} x {n:12,d} = {ninst*n:14,d}  samples {smp}")

if "--stalls" in sys.argv:
    # top instructions per stall reason
    reasons = ["stall_long_sb", "stall_wait", "stall_no_inst", "stall_math", "stall_dispatch", "stall_branch_resolving", "stall_short_sb", "stall_lg"]
    for rs in reasons:
        if rs not in ix:
            continue
        tot_r = 0; items = []
        for r in data:
            try:
                v = int(r[ix[rs]])
            except Exception:
                continue
            tot_r += v
            items.append((v, r[ix["Address"]][-5:], r[ix["Source"]].strip()[:70]))
        items.sort(reverse=True)
        print(f"== {rs}: {tot_r}")
        for v, a, s in items[:6]:
            print(f"   {v:7d} {a} {s}")
