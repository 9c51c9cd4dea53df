"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py rep  <report.ncu-rep> <label> [algorithmic_bytes_per_launch]
    python tools/ncu_summary.py list <launches.csv> <label>
Appends a markdown section to profiles/<round>_ncu.md and updates profiles/traffic.json.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(REPO, "profiles")
KEYS = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "smsp__inst_executed.sum",
        "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum", "nvlrx__bytes.sum", "nvltx__bytes.sum"]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1, "nsecond": 1e-9}


def rep(path, label, alg=None, round_tag="r1"):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"\n## {label}\n", f"source: `{os.path.basename(path)}` (ncu --set full --clock-control none)\n",
             "| metric | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " |",
             "|---|" + "---|" * (len(rows) - 2)]
    vals = {}
    for k in KEYS:
        if k not in hdr:
            continue
        j = hdr.index(k)
        cells = [r[j] for r in rows[2:]]
        lines.append(f"| {k} ({units[j]}) | " + " | ".join(c[:70] for c in cells) + " |")
        vals[k] = [(c, units[j]) for c in cells]
    traffic = []
    for i in range(len(rows) - 2):
        try:
            rd = float(vals["dram__bytes_read.sum"][i][0].replace(",", "")) * SCALE[vals["dram__bytes_read.sum"][i][1]]
            wr = float(vals["dram__bytes_write.sum"][i][0].replace(",", "")) * SCALE[vals["dram__bytes_write.sum"][i][1]]
            t = float(vals["gpu__time_duration.sum"][i][0].replace(",", "")) * SCALE[vals["gpu__time_duration.sum"][i][1]]
            traffic.append((rd + wr, t))
        except (KeyError, ValueError):
            pass
    if traffic:
        tb, t = traffic[-1]
        lines.append(f"\ntraffic per launch (dram read+write): {tb / 1e6:.1f} MB; duration {t * 1e6:.1f} us"
                     + (f"; algorithmic bytes {alg / 1e6:.1f} MB -> traffic/algorithmic = {tb / alg:.3f}"
                        f", achieved {alg / t / 1e9:.1f} GB/s (cold, serialised)" if alg else ""))
        tj = os.path.join(PROF, "traffic.json")
        d = json.load(open(tj)) if os.path.exists(tj) else {}
        d[label] = {"traffic_bytes_per_launch": tb, "algorithmic_bytes_per_launch": alg,
                    "duration_s": t, "report": os.path.basename(path), "round": round_tag}
        json.dump(d, open(tj, "w"), indent=1)
    with open(os.path.join(PROF, f"{round_tag}_ncu.md"), "a") as f:
        f.write("\n".join(lines) + "\n")


def launch_list(path, label, round_tag="r1"):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    idx = {k: j for j, k in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = SCALE.get(r[idx["Metric Unit"]], 1e-9)
        name = r[idx["Kernel Name"]]
        agg[name][0] += 1
        agg[name][1] += float(r[idx["Metric Value"]].replace(",", "")) * unit
    tot = sum(v[1] for v in agg.values())
    lines = [f"\n## launch list: {label}\n", f"source: `{os.path.basename(path)}` "
             "(ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)\n",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k[:90]}` | {n} | {v * 1e3:.2f} | {v / tot * 100:.1f}% |")
    with open(os.path.join(PROF, f"{round_tag}_ncu.md"), "a") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    os.makedirs(PROF, exist_ok=True)
    rt = os.environ.get("ROUND_TAG", "r1")
    if sys.argv[1] == "rep":
        rep(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None, rt)
    else:
        launch_list(sys.argv[2], sys.argv[3], rt)
