"""Instruction mix (per amplitude) and stall samples per opcode for each
kernel in an ncu SASS source export: python scripts/sass_mix.py src.csv [amps]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
amps = float(sys.argv[2]) if len(sys.argv) > 2 else 2 ** 27
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
        continue
    cur.append(r)
for bi, b in enumerate(blocks[::2]):
    h = b[0]
    ie, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    mix, stall, tot, stot = collections.Counter(), collections.Counter(), 0, 0
    for r in b[1:]:
        n = int(r[ie] or 0)
        if not n:
            continue
        toks = r[1].split()
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        mix[op] += n
        tot += n
        stall[op] += int(r[si] or 0)
        stot += int(r[si] or 0)
    print(f"kernel {bi}: {tot} warp-inst, {tot * 32 / amps:.1f} per amplitude, {stot} stall samples")
    for k, v in mix.most_common(22):
        print(f"  {k:8s} {100 * v / tot:5.1f}%  per-amp {v * 32 / amps:6.2f}  stall {100 * stall[k] / max(stot, 1):5.1f}%")
