"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

python tools/launch_list.py gpurun_out/<tag>_launches.csv --out profiles/<tag>_launch_list.md [--title ...]
"""
import argparse
import csv
import io
import re
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="launch list")
    ap.add_argument("--command", default="")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    text = open(a.csv).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ms = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1.0)
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        tot[name] += ms
        cnt[name] += 1
    total = sum(tot.values())
    lines = [f"# {a.title}", ""]
    if a.command:
        lines += [f"Command: `{a.command}`", ""]
    lines += ["Per-launch times are serialised and cold-cache (ncu), so only the shares compare with "
              "bench.py's CUDA-event breakdown.",
              f"Kernels profiled: {sum(cnt.values())} launches, total {total:.2f} ms.", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for name, ms in sorted(tot.items(), key=lambda kv: -kv[1])[:a.top]:
        lines.append(f"| `{name}` | {cnt[name]} | {ms:.3f} | {100 * ms / total:.1f}% |")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    main()
