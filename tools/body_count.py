"""Instructions in the innermost ACS loop body of a kernel's SASS (the loop holding the most
VIADDMNMX.U16x2), by opcode: python tools/body_count.py <obj.o|lib.so> <kernel> [n]"""
import collections
import re
import subprocess
import sys


def body(obj, fn):
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
    ins = [(int(m.group(1), 16), m.group(2).strip()) for m in
           (re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln) for ln in sass.splitlines()) if m]
    best = None
    for a, i in ins:
        m = re.search(r"BRA\s+(?:!?U?P\d, )?0x([0-9a-f]+)", i)
        if m and int(m.group(1), 16) < a:
            t = int(m.group(1), 16)
            span = [j for b, j in ins if t <= b <= a]
            n = sum("VIADDMNMX.U16x2" in j for j in span)
            if best is None or (n, -len(span)) > (best[0], -len(best[1])):
                best = (n, span)
    return best[1]


def op(i):
    x = i.split()
    return x[1] if x[0].startswith("@") else x[0]


if __name__ == "__main__":
    b = body(sys.argv[1], sys.argv[2])
    c = collections.Counter(op(i) for i in b)
    print(sys.argv[1], sys.argv[2], "body instructions:", len(b))
    for k, v in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 12):
        print(f"  {k:24s}{v}")
