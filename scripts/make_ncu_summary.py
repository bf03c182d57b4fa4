"""Summarise `ncu --set full` raw-page CSV exports of the dominant QFT sweeps
into profiles/:
  * <tag>_k_qft_<dtype>.txt : duration, DRAM bytes, pipe utilisation,
    occupancy, bank conflicts and the top pc-sampling stall reasons per launch;
  * ncu_summary.json         : DRAM bytes per launch per workload, stamped with
    the sha256 of the libshardcu.so that was profiled — bench.py reports it as
    roofline.traffic only when the loaded library has the same hash.

    python scripts/make_ncu_summary.py <tag> qft27_c128=<raw.csv> [qft27_c64=<raw.csv> ...]
"""
import csv
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2304_14969_b200 import _build  # noqa: E402
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarise(path: Path):
    rows = list(csv.reader(io.StringIO(path.read_text())))
    h, units = rows[0], rows[1]
    lines, per_launch = [], []
    for r in rows[2:]:
        lines.append(f"kernel: {r[h.index('Kernel Name')]}")
        for k in KEYS:
            if k in h:
                lines.append(f"  {k:62s} {r[h.index(k)]:>18s} {units[h.index(k)]}")
        stalls = [(h[i], float(r[i] or 0)) for i in range(len(h))
                  if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued")]
        tot = sum(v for _, v in stalls) or 1
        lines.append("  stall reasons (pc sampling):")
        for k, v in sorted(stalls, key=lambda x: -x[1])[:8]:
            lines.append(f"    {v / tot * 100:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
        rd = float(r[h.index("dram__bytes_read.sum")]) * SCALE[units[h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")]) * SCALE[units[h.index("dram__bytes_write.sum")]]
        per_launch.append(rd + wr)
    return lines, per_launch


def main():
    tag = sys.argv[1]
    lib = ROOT / "paper_2304_14969_b200" / "libshardcu.so"
    out = {"tag": tag, "kqft_sass_sha256": _build.kernel_sass_sha256("k_qft", lib),
           "so_sha256": _build.device_code_sha256(lib), "so_sha256_of": ".nv_fatbin section", "captures": {}}
    for arg in sys.argv[2:]:
        name, _, path = arg.partition("=")
        lines, per = summarise(Path(path))
        (ROOT / "profiles" / f"{tag}_k_qft_{name}.txt").write_text("\n".join(lines) + "\n")
        out["captures"][name] = {"source": Path(path).name, "dram_bytes_per_launch": sum(per) / len(per),
                                 "dram_bytes_each": per}
    (ROOT / "profiles" / "ncu_summary.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
