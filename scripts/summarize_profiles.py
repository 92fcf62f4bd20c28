"""Summaries of the ncu captures made by scripts/profile_round1.sh (run here, on the files
gpurun brought back):

  profiles/<round>/launch_summary.txt   per-kernel share of the launch list (timed region)
  profiles/<round>/ncu_full_summary.txt per-launch DRAM traffic, duration, L2 hit rate, ...
  profiles/<round>/traffic.json         per-kernel DRAM bytes per launch (bench.py roofline.traffic)

usage: python scripts/summarize_profiles.py gpurun_out profiles/round1
"""
import collections
import csv
import io
import re
import json
import os
import shutil
import subprocess
import sys


def kname(full):
    """kernel name without the parameter list; template casts like (int)0 are dropped first"""
    return re.sub(r"\((?:int|bool|unsigned int)\)", "", full).split("(")[0].strip()


def launch_summary(csv_path, out_path, cmd):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0.0, 0])
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit == "us" else v if unit == "ms" else v * 1e3
        name = kname(r[ik])
        agg[name][0] += ms
        agg[name][1] += 1
    total = sum(a[0] for a in agg.values())
    n = sum(a[1] for a in agg.values())
    with open(out_path, "w") as fh:
        fh.write("ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off\n")
        fh.write(f"command: {cmd}\n")
        fh.write("per-launch times are cold-cache and serialised: compare SHARES\n")
        fh.write(f"total launches {n}, total {total:.2f} ms\n")
        for name, (ms, cnt) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
            fh.write(f"{100 * ms / total:6.2f}%  {ms:10.3f} ms  {cnt:5d} launches  {ms / cnt:9.4f} ms/launch  {name}\n")
    return agg


def full_summary(reps, out_txt, out_json):
    """reps: list of (title, path); a path is an .ncu-rep (read with ncu -i) or a raw-page CSV
    exported on the GPU box (scripts/profile_round2.sh)"""
    traffic = collections.defaultdict(list)
    with open(out_txt, "w") as fh:
        fh.write("ncu --set full --clock-control none (raw page, demangled names); DRAM bytes and durations per launch\n")
        for title, path in reps:
            if not os.path.exists(path):
                continue
            fh.write(f"\n== {title} ({os.path.basename(path)})\n")
            _one_report(path, fh, traffic)
    json.dump({k: {"dram_bytes_per_launch": sum(v) / len(v), "launches_captured": len(v)} for k, v in traffic.items()},
              open(out_json, "w"), indent=1)


def _one_report(rep, fh, traffic):
    if rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-kernel-base", "demangled"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
    idx = {w: hdr.index(w) for w in want if w in hdr}

    def val(r, w):
        i = idx.get(w)
        if i is None or not r[i]:
            return None
        x = float(r[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1,
                 "s": 1e3}.get(u, 1)
        return x * scale

    if True:
        fh.write("kernel | duration ms | DRAM read MB | DRAM write MB | DRAM GB/s | L2 hit % | regs | grid x block\n")
        for r in rows[2:]:
            if len(r) != len(hdr):
                continue
            name = kname(r[hdr.index("Kernel Name")])
            d = val(r, "gpu__time_duration.sum")
            rd = val(r, "dram__bytes_read.sum") or 0.0
            wr = val(r, "dram__bytes_write.sum") or 0.0
            gbs = (rd + wr) / (d * 1e-3) / 1e9 if d else 0.0
            grid = int(val(r, 'launch__grid_size') or 0)
            traffic[f"{name} grid {grid}"].append(rd + wr)
            fh.write(f"{name} | {d:.4f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {gbs:.1f} | "
                     f"{val(r, 'lts__t_sector_hit_rate.pct') or 0:.1f} | "
                     f"{int(val(r, 'launch__registers_per_thread') or 0)} | "
                     f"{grid} x {int(val(r, 'launch__block_size') or 0)}\n")


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    cmd = "PMG_PROFILE_REGION=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline  (config 5, ILUT, one timed " \
          "solve)"
    launch_summary(os.path.join(src, "launches.csv"), os.path.join(dst, "launch_summary.txt"), cmd)
    shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, "launches_config5_ilut_solve.csv"))
    j = lambda f: os.path.join(src, f)
    full = j("prof_full_raw.csv") if os.path.exists(j("prof_full_raw.csv")) else j("prof_full.ncu-rep")
    full_summary([("config 5 ILUT solve: first launches of every kernel of one V-cycle", full),
                  ("config 5 Gauss-Seidel solve: upper-sum pre-pass, GS sweep", j("gs_full_raw.csv")),
                  ("setup on config 3: GPU assembly kernels, GPU ILUT", j("setup_full_raw.csv"))],
                 os.path.join(dst, "ncu_full_summary.txt"), os.path.join(dst, "traffic.json"))
    if os.path.exists(os.path.join(src, "prof_plain.json")):
        shutil.copy(os.path.join(src, "prof_plain.json"), os.path.join(dst, "bench_line_under_profile_region.json"))


if __name__ == "__main__":
    main()
