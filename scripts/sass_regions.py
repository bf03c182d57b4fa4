"""Group an ncu SASS source export (first kernel) into straight-line regions
and print the most expensive ones (instructions per warp, stall samples)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
warps = float(sys.argv[2]) if len(sys.argv) > 2 else 2 ** 14 * 16
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
        continue
    cur.append(r)
b = blocks[which]
h = b[0]
si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
lines = []
for r in b[1:]:
    try:
        n, s = int(r[ie] or 0), int(r[si] or 0)
    except ValueError:
        continue
    lines.append((r[0][-5:], n, s, r[1].strip()[:60]))
groups = []
for a, n, s, t in lines:
    if groups and groups[-1][1] == n:
        groups[-1][2] += 1
        groups[-1][3] += s
        groups[-1][5] = t
    else:
        groups.append([a, n, 1, s, t, t])
print("instr per warp", sum(n for _, n, _, _ in lines) / warps, "samples", sum(s for _, _, s, _ in lines))
for g in sorted(groups, key=lambda g: -g[1] * g[2])[:int(sys.argv[4]) if len(sys.argv) > 4 else 18]:
    print(f"{g[0]} x{g[1]/warps:6.1f} n={g[2]:4d} tot={g[1]*g[2]/warps:7.1f} stall={g[3]:6d}  {g[4]} ... {g[5]}")
