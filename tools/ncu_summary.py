"""Summarise an ncu launch list + --set full capture into profiles/.

    python tools/ncu_summary.py <launches.csv> <prof.ncu-rep> <tag>

Writes profiles/ncu_<tag>.md (human summary) and profiles/ncu_summary.json
(per-kernel DRAM bytes per launch, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "B": 1}


def short(name: str) -> str:
    for key in ("ffa_fwd", "ffa_bwd_dkdv", "ffa_bwd_dq", "bwd_preprocess", "range_gather",
                "range_scatter", "cast"):
        if key in name:
            return key
    return name[:40]


def launches(path: Path):
    rows = [r for r in csv.reader(io.StringIO("".join(l for l in path.read_text().splitlines(True)
                                                       if not l.startswith("==")))) if r]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    out = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "ns"
        ms = v / 1e6 if unit in ("ns", "nsecond") else (v / 1e3 if unit in ("us", "usecond") else v)
        out.append((short(r[ki]), ms))
    return out


def full(path: Path):
    txt = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    val = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if m.startswith("dram__bytes"):
                    val *= SCALE.get(units[i], 1)
                d[m] = val
                d[m + ".unit"] = units[i]
        res.append(d)
    return res


def main():
    lpath, fpath, tag = Path(sys.argv[1]), Path(sys.argv[2]), sys.argv[3]
    ls = launches(lpath)
    fl = full(fpath)
    total = {}
    for k, ms in ls:
        total.setdefault(k, []).append(ms)
    step = sum(statistics.mean(v) for v in total.values())
    md = [f"# ncu summary {tag}", "", "Launch list (`--metrics gpu__time_duration.sum "
          "--clock-control none`, cold-cache, serialised):", "",
          "| kernel | launches | mean ms | share of step |", "|---|---|---|---|"]
    for k, v in total.items():
        md.append(f"| {k} | {len(v)} | {statistics.mean(v):.3f} | {statistics.mean(v) / step:.1%} |")
    md += ["", "`--set full` capture (one launch each):", "",
           "| kernel | ms | DRAM read | DRAM write | tensor pipe active % | SM throughput % | regs | warps active % |",
           "|---|---|---|---|---|---|---|---|"]
    summ = {"tag": tag, "dram_bytes_per_launch": {}, "launch_share": {}}
    for d in fl:
        rd = d.get("dram__bytes_read.sum", 0.0)
        wr = d.get("dram__bytes_write.sum", 0.0)
        summ["dram_bytes_per_launch"][d["kernel"]] = rd + wr
        md.append(f"| {d['kernel']} | {d.get('gpu__time_duration.sum', 0):.3f} "
                  f"{d.get('gpu__time_duration.sum.unit', '')} | {rd / 1e6:.1f} MB | {wr / 1e6:.1f} MB | "
                  f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                  f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                  f"{d.get('launch__registers_per_thread', 0):.0f} | "
                  f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} |")
    for k, v in total.items():
        summ["launch_share"][k] = statistics.mean(v) / step
    (ROOT / "profiles" / f"ncu_{tag}.md").write_text("\n".join(md) + "\n")
    (ROOT / "profiles" / "ncu_summary.json").write_text(json.dumps(summ, indent=1) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
