"""Summarise an ncu SASS source page (csv): top instructions by stall samples, totals by opcode."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iss, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((r[ia], r[isrc], int(r[iss] or 0), int(r[iex] or 0)))
    except (ValueError, IndexError):
        pass
tot_s = sum(d[2] for d in data); tot_e = sum(d[3] for d in data)
print("samples", tot_s, "warp instr", tot_e)
op = collections.Counter(); ops = collections.Counter()
for a, s, n, e in data:
    o = s.split()[0] if s.split() else "?"
    if o.startswith("@"):
        o = s.split()[1]
    o = o.split(".")[0]
    op[o] += e; ops[o] += n
print("by opcode (instr%, samples%):")
for o, e in op.most_common(30):
    print(f"  {o:10s} {100*e/tot_e:5.1f} {100*ops[o]/tot_s:5.1f}")
k = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print("top instructions by samples:")
for a, s, n, e in sorted(data, key=lambda d: -d[2])[:k]:
    print(f"  {a} {n:6d} {e:9d}  {s[:90]}")
