"""Summarise an ncu launch list + a full capture of the sweep kernel into
profiles/ (tracked): per-kernel time shares, dram traffic, pipe use."""
import collections
import csv
import json
import subprocess
import sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    for d in data:
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", "nsecond"), 1e-6)
            name = d["Kernel Name"].split("(")[0]
            agg[name][0] += 1
            agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": c, "ms": v, "share": v / tot} for k, (c, v) in
            sorted(agg.items(), key=lambda x: -x[1][1])]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def main(launch_csv, rep, out_json, algorithmic_bytes, tag):
    L = launches(launch_csv)
    d, u = raw(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
            "smsp__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum", "lts__t_bytes.sum"]
    m = {k: (d.get(k), u.get(k)) for k in keys}
    gb = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    traffic = sum(float(d[k]) * gb.get(u[k], 1.0) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    # warp stall reasons (all warps of the sweep, cycles per issued instruction)
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
              for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    stalls = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    summary = {"tag": tag, "launch_list": L, "sweep_full_capture": m, "sweep_stall_cycles_per_issue": stalls,
               "sweep_dram_bytes_per_launch": traffic, "sweep_algorithmic_bytes": algorithmic_bytes,
               "traffic_over_algorithmic": traffic / algorithmic_bytes if algorithmic_bytes else None}
    json.dump(summary, open(out_json, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:2500])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]), sys.argv[5])
