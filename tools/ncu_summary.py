"""Summarise `ncu --set full` reports into profiles/ (markdown + traffic json).

python tools/ncu_summary.py <tag=rep> ... --out profiles/r1_ncu.md
Each positional argument is "<layer tags comma-separated>=<path.ncu-rep>"; the
kernels of a report are matched to the tags in launch order, skipping the
small split-K reduction and weight-packing launches, or explicitly as
"tag@index,..." (index = launch order inside the report).  Writes the per-kernel key metrics and
profiles/ncu_traffic.json {tag: {"kernel", "dram_bytes", "duration_ms"}}.
"""
import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (active)"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, u, v in zip(hdr, units, r)} for r in rows[2:]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu --set full summary")
    a = ap.parse_args()
    md = [f"# {a.title}", "", "Command: `tools/profile_round.sh` (ncu --set full --clock-control none "
          "--import-source on --nvtx, one GPU, kernels selected by NVTX layer range).", ""]
    traffic_path = Path(a.out).parent / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    for spec in a.reports:
        tags, rep = spec.split("=", 1)
        allk = raw(rep)
        if "@" in tags:  # explicit "tag@launch-index" list
            pairs = [(t.split("@")[0], allk[int(t.split("@")[1])]) for t in tags.split(",")]
        else:
            kernels = [k for k in allk if not any(s in k["Kernel Name"][0] for s in ("reduce_part", "pack_"))]
            pairs = list(zip(tags.split(","), kernels))
        for tag, k in pairs:
            name = k["Kernel Name"][0]
            md.append(f"## {tag}: `{name[:110]}`")
            md.append("")
            md.append("| metric | value |")
            md.append("|---|---|")
            vals = {}
            for key, label in KEYS:
                if key in k:
                    v, u = k[key]
                    md.append(f"| {label} (`{key}`) | {v} {u} |")
                    vals[key] = (v, u)
            md.append("")
            rd, ur = vals.get("dram__bytes_read.sum", ("0", "byte"))
            wr, uw = vals.get("dram__bytes_write.sum", ("0", "byte"))
            db = float(rd.replace(",", "")) * SCALE.get(ur, 1) + float(wr.replace(",", "")) * SCALE.get(uw, 1)
            dur, udur = vals.get("gpu__time_duration.sum", ("0", "ms"))
            ms = float(dur.replace(",", "")) * {"ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}.get(udur, 1)
            traffic[tag] = {"kernel": name[:160], "dram_bytes": db, "duration_ms": ms, "report": Path(rep).name}
    Path(a.out).write_text("\n".join(md) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")


if __name__ == "__main__":
    main()
