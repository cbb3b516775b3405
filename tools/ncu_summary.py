"""Summarise ncu output for profiles/ (run here, on the CPU side, after a gpurun
call brought the reports back into gpurun_out/).

  python tools/ncu_summary.py --tag r01 \
      --launches gpurun_out/launches_r01.csv --full gpurun_out/prof_r01_full.ncu-rep

writes profiles/<tag>_launches.md (per-kernel launch statistics of the
`--metrics gpu__time_duration.sum` pass) and profiles/<tag>_ncu_full.{md,json}
(selected metrics of the `--set full` capture: duration, DRAM bytes, throughput,
registers, warp stall breakdown).  bench.py reads the JSON's DRAM bytes for the
roofline `traffic` field."""
import argparse
import collections
import csv
import io
import json
import os
import statistics
import subprocess

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_pct_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "smem_dyn"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("smsp__inst_executed.sum", "inst_executed"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
              "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}


def launches(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    per = collections.defaultdict(list)
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", "")) * UNIT_SCALE.get(r["Metric Unit"], 1.0)
        per[r["Kernel Name"].split("(")[0]].append(v)      # microseconds
    return per


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, key in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[key] = v * UNIT_SCALE.get(units[i], 1.0)
        stalls = {}
        for i, h in enumerate(hdr):
            p = "smsp__average_warps_issue_stalled_"
            if h.startswith(p) and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls[h[len(p):-len("_per_issue_active.ratio")]] = float(r[i])
                except ValueError:
                    pass
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        # tensor-pipe utilisation (legacy HMMA and tcgen05 pipes): every raw
        # metric of the capture that names the tensor pipe, as reported
        tp = {}
        for i, h in enumerate(hdr):
            if ("pipe_tensor" in h or "pipe_tc" in h or "tcgen05" in h or "utc" in h.lower()) and \
                    ("pct" in h or h.endswith(".sum") or h.endswith(".avg")):
                try:
                    tp[h] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        d["tensor_pipe"] = tp
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--note", default="")
    ap.add_argument("--k2pair", help="JSON from tools/ncu_k2pair.py: algorithmic bytes of the "
                                     "captured K2a + K2b launch pair")
    a = ap.parse_args()
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
    if a.launches:
        per = launches(a.launches)
        tot = sum(sum(v) for v in per.values())
        with open(os.path.join(root, f"{a.tag}_launches.md"), "w") as f:
            f.write(f"# {a.tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
            f.write("Cold-cache, serialised per-launch times; compare SHARES with bench.py, "
                    "not absolutes.\n\n")
            if a.note:
                f.write(a.note + "\n\n")
            f.write("| kernel | launches | mean us | median us | min us | max us | share |\n")
            f.write("|---|---|---|---|---|---|---|\n")
            for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"| {k} | {len(v)} | {statistics.mean(v):.2f} | {statistics.median(v):.2f}"
                        f" | {min(v):.2f} | {max(v):.2f} | {sum(v) / tot:.3f} |\n")
    if a.full:
        res = full(a.full)
        with open(os.path.join(root, f"{a.tag}_ncu_full.json"), "w") as f:
            json.dump({"source": os.path.basename(a.full), "note": a.note, "kernels": res}, f,
                      indent=1)
        with open(os.path.join(root, f"{a.tag}_ncu_full.md"), "w") as f:
            f.write(f"# {a.tag}: ncu --set full capture ({os.path.basename(a.full)})\n\n")
            if a.note:
                f.write(a.note + "\n\n")
            for d in res:
                f.write(f"## {d['kernel']}\n\n")
                for m, key in FULL_METRICS:
                    if key in d:
                        f.write(f"- {key} ({m}): {d[key]:,.3f}\n")
                if "duration" in d and "dram_read" in d:
                    gbs = (d["dram_read"] + d.get("dram_write", 0)) / (d["duration"] * 1e-6) / 1e9
                    f.write(f"- DRAM GB/s over the launch: {gbs:,.1f}\n")
                f.write(f"- top stalls (warps per issue): {d['stalls_per_issue']}\n")
                if d.get("tensor_pipe"):
                    f.write(f"- tensor pipe: {d['tensor_pipe']}\n")
                f.write("\n")
        if a.k2pair:
            with open(a.k2pair) as f:
                alg = json.load(f)
            pair = [d for d in res if "gemv_kernel" in d["kernel"]][:2]
            dram = sum(d["dram_read"] + d.get("dram_write", 0.0) for d in pair)
            dur = sum(d["duration"] for d in pair)
            out = {"kernels": [d["kernel"] for d in pair], "dram_bytes": dram,
                   "alg_bytes": alg["alg_bytes"], "alg_detail": alg,
                   "duration_us_serialised": dur,
                   "note": "one K2a + K2b launch pair of one known forward (same decisions every "
                           "repeat), ncu --set full; DRAM bytes vs that forward's algorithmic bytes"}
            with open(os.path.join(root, f"{a.tag}_k2pair.json"), "w") as f:
                json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
