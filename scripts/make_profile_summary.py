"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked):
  profiles/<tag>_launches.csv      per-launch device times (ncu launch list)
  profiles/<tag>_k_qft.txt       full-set metrics of the k_qft launches
  profiles/ncu_summary.json        DRAM bytes per sweep launch (bench.py `traffic`)
usage: python scripts/make_profile_summary.py <tag> [prof.ncu-rep] [launches.csv] [bench.json]"""
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
rep = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "gpurun_out" / "prof_raw.csv"
launches = Path(sys.argv[3]) if len(sys.argv) > 3 else ROOT / "gpurun_out" / "launches.csv"
bench = Path(sys.argv[4]) if len(sys.argv) > 4 else ROOT / "gpurun_out" / "bench.json"
out = ROOT / "profiles"
out.mkdir(exist_ok=True)

if rep.suffix == ".csv":  # raw page exported on the GPU box
    raw = rep.read_text()
else:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
lines, dram = [], []
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    lines.append(f"kernel: {name}")
    for k in keys:
        if k in h:
            lines.append(f"  {k:62s} {r[h.index(k)]:>16s} {units[h.index(k)]}")
    stalls = [(h[i], float(r[i] or 0)) for i in range(len(h))
              if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued")]
    tot = sum(v for _, v in stalls) or 1
    lines.append("  stall reasons (pc sampling):")
    for k, v in sorted(stalls, key=lambda x: -x[1])[:8]:
        lines.append(f"    {v / tot * 100:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
    rd = float(r[h.index("dram__bytes_read.sum")]) * (1e9 if units[h.index("dram__bytes_read.sum")] == "Gbyte" else 1e6)
    wr = float(r[h.index("dram__bytes_write.sum")]) * (1e9 if units[h.index("dram__bytes_write.sum")] == "Gbyte" else 1e6)
    dram.append(rd + wr)
(out / f"{tag}_k_qft.txt").write_text("\n".join(lines) + "\n")
summary = {"tag": tag, "source": str(rep.name), "dram_bytes_per_sweep": sum(dram) / len(dram),
           "dram_bytes_per_launch": dram}
if bench.exists():
    try:
        b = json.loads(bench.read_text().strip().splitlines()[-1])
        summary["bench_ms_per_step"] = b.get("ms_per_step")
        summary["bench_roofline"] = b.get("roofline")
    except Exception:
        pass
(out / "ncu_summary.json").write_text(json.dumps(summary, indent=1) + "\n")
if launches.exists():
    shutil.copy(launches, out / f"{tag}_launches.csv")
print((out / f"{tag}_k_qft.txt").read_text())
print(json.dumps(summary, indent=1))
