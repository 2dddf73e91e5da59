"""Per-opcode and per-stall breakdown of an ncu source-page export
(`ncu -i rep --page source --csv --print-source sass`): executed warp
instructions by opcode and stall samples by opcode, for the hot loop.
Usage: python profiles/sass_hot.py src.csv [min_exec]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
minx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ops = collections.Counter()
st = collections.defaultdict(collections.Counter)
tot = 0
for r in rows[2:]:
    ex = int(r[ix["Instructions Executed"]] or 0)
    if ex < minx:
        continue
    src = r[ix["Source"]].strip()
    tok = src.split()
    op = tok[1] if tok and tok[0].startswith("@") else (tok[0] if tok else "?")
    op = op.rstrip(",")
    ops[op] += ex
    tot += ex
    for k in h:
        if k.startswith("stall_") and "Not Issued" not in k:
            st[op][k[6:]] += int(r[ix[k]] or 0)
print("total warp-instr", tot)
for op, n in ops.most_common(40):
    s = st[op]
    top = ", ".join(f"{k}={v}" for k, v in s.most_common(4) if v)
    print(f"{op:28s} {n:>12d} {n / tot:6.3f}  {top}")
agg = collections.Counter()
for s in st.values():
    agg.update(s)
print("stalls:", ", ".join(f"{k}={v}" for k, v in agg.most_common(10)))
