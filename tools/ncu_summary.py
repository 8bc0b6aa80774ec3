"""Summarise ncu reports (gpurun_out/*.ncu-rep, launch-list CSVs) into profiles/.

    python tools/ncu_summary.py <out_dir> <rep1.ncu-rep> [...] [--launches launches.csv]

Writes <out_dir>/ncu_summary.json (per kernel: duration, tensor-pipe %, DRAM bytes,
L2->SM bytes, top stall reasons) and <out_dir>/launch_shares.txt (kernel time shares
from the gpu__time_duration launch list; cold-cache, serialised: compare shares only).
"""
import csv
import json
import os
import subprocess
import sys
import collections

KEYS = {
    "duration_ms": ("gpu__time_duration.sum", {"ms": 1, "us": 1e-3, "s": 1e3, "ns": 1e-6}),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", None),
    "dram_read_bytes": ("dram__bytes_read.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
    "dram_write_bytes": ("dram__bytes_write.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
    "l2_to_sm_bytes": ("l1tex__m_xbar2l1tex_read_bytes.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
    "grid": ("launch__grid_size", None),
    "block": ("launch__block_size", None),
    "registers": ("launch__registers_per_thread", None),
    "sm_mhz": ("sm__cycles_elapsed.avg.per_second", {"cycle/second": 1e-6, "cycle/nsecond": 1e3, "cycle/usecond": 1}),
}


def _f(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def summarise_rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
    res = {"kernel": d.get("Kernel Name", "")}
    for k, (m, conv) in KEYS.items():
        if m in d:
            v = _f(d[m])
            if conv and v is not None:
                v *= conv.get(u.get(m, ""), 1)
            res[k] = v
    res["dram_bytes"] = (res.get("dram_read_bytes") or 0) + (res.get("dram_write_bytes") or 0)
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): _f(v)
              for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    res["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -(kv[1] or 0))[:5])
    return res


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[mi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'launches':>8} {'ms':>9} {'share':>6}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v[0]:8d} {v[1] / 1e6:9.3f} {100 * v[1] / tot:5.1f}%  {k}")
    lines.append(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
    return "\n".join(lines)


if __name__ == "__main__":
    out_dir = sys.argv[1]
    os.makedirs(out_dir, exist_ok=True)
    args = sys.argv[2:]
    summ = {}
    if "--launches" in args:
        i = args.index("--launches")
        with open(os.path.join(out_dir, "launch_shares.txt"), "w") as f:
            f.write(launch_shares(args[i + 1]) + "\n")
        args = args[:i] + args[i + 2:]
    traffic_out = None
    if "--traffic" in args:
        i = args.index("--traffic")
        traffic_out = args[i + 1]
        args = args[:i] + args[i + 2:]
    for rep in args:
        s = summarise_rep(rep)
        summ[os.path.basename(rep)] = s
    if traffic_out:
        # per-launch DRAM bytes keyed by the kernel's short name (bench.py's roofline traffic)
        tr = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum of one captured launch per kernel "
                       "(ncu --set full --clock-control none), C2 B=1024 S=1024 bf16; see ncu_summary.json"}
        for rep, v in summ.items():
            short = v["kernel"].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
            tr[short] = {"dram_bytes_per_launch": v.get("dram_bytes"), "launch": "one launch per step (%s)" % rep,
                         "duration_ms_under_ncu": v.get("duration_ms"), "tensor_pipe_pct": v.get("tensor_pipe_pct")}
        with open(traffic_out, "w") as f:
            json.dump(tr, f, indent=1)
    with open(os.path.join(out_dir, "ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ, indent=1)[:3000])
