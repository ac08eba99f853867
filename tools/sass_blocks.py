"""Hot straight-line blocks of one kernel from an ncu SASS source CSV.
usage: python tools/sass_blocks.py sass.csv N_INSTANCES [top] [dump_addr_suffix...]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
dump = set(sys.argv[4:])
h = rows[1]
ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
ist = h.index("Warp Stall Sampling (All Samples)")
seq = [(r[ia][-5:], r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)) for r in rows[2:] if len(r) > iex]
blocks, cur = [], None
for a, s, e, st in seq:
    if cur is None or e != cur[2]:
        cur = [a, [], e, 0]
        blocks.append(cur)
    cur[1].append((a, s, st))
    cur[3] += st
for b in sorted(blocks, key=lambda b: -len(b[1]) * b[2])[:top]:
    print(f"{b[0]} len {len(b[1]):4d} exec/inst {b[2] / n:6.2f} contrib {len(b[1]) * b[2] / n:7.1f} stall {b[3]}")
for b in blocks:
    if b[0] in dump:
        print(f"---- {b[0]} exec/inst {b[2] / n:.2f}")
        for a, s, st in b[1]:
            print(f"  {a} {st:6d} {s}")
