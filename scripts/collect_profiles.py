#!/usr/bin/env python
"""Copy the evidence produced by scripts/gpu_final_check.sh (gpurun_out/prof)
into profiles/ under a round prefix, summarise the ncu reports, and update
profiles/traffic.json from the full captures.

    python scripts/collect_profiles.py r02
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")


def last_json(path):
    lines = [l for l in open(path).read().splitlines() if l.startswith("{")]
    return lines[-1] if lines else None


def dram(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki = h.index("Kernel Name")
    ri, wi = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    unit = rows[1][ri]
    mul = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}[unit]
    res = {}
    for r in rows[2:]:
        name = r[ki].split("(")[0].split("::")[-1].split("<")[0]
        res.setdefault(name, int((float(r[ri]) + float(r[wi])) * mul))
    return res


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    copies = {"bench_wan.json": "bench_wan.json", "bench_cog.json": "bench_cog.json",
              "bench_wan_gt.json": "bench_wan_asa_gt.json", "bench_ref.json": "bench_reference_arm.json",
              "bench_bwd_wan.json": "bench_bwd_wan.json", "bench_bwd_cog.json": "bench_bwd_cog.json",
              "bench_bwd_wan_asa_gt.json": "bench_bwd_wan_asa_gt.json",
              "bench_bwd_cog_asa_gt.json": "bench_bwd_cog_asa_gt.json",
              "launches_wan.csv": "launches_wan_keep51.csv", "launches_cog.csv": "launches_cog_keep25.csv",
              "launches_bwd_wan.csv": "launches_bwd_wan.csv", "sweep_wan.jsonl": "sweep_wan.jsonl",
              "pytest_gpu.log": "pytest_gpu.log", "smoke.log": "smoke.log",
              "bench_wan_200.json": "bench_wan_sustained200.json",
              "bench_wan_tau.json": "bench_wan_tau0.9.json",
              "mask_time_wan.jsonl": "mask_time_wan.jsonl", "mask_time_cog.jsonl": "mask_time_cog.jsonl",
              "pipes_wan.csv": "pipes_wan_keep51.csv", "pipes_cog.csv": "pipes_cog_keep25.csv",
              "pipes_wan_tau95.csv": "pipes_wan_tau0.95.csv",
              "sanitizer_memcheck.log": "sanitizer_memcheck.log",
              "sanitizer_racecheck.log": "sanitizer_racecheck.log",
              "sanitizer_synccheck.log": "sanitizer_synccheck.log"}
    for s, d in copies.items():
        p = os.path.join(SRC, s)
        if os.path.exists(p):
            if s.endswith(".json"):
                line = last_json(p)
                if line:
                    open(os.path.join(DST, f"{tag}_{d}"), "w").write(line + "\n")
            else:
                shutil.copy(p, os.path.join(DST, f"{tag}_{d}"))
    traffic = {"_note": "dram__bytes_read.sum + dram__bytes_write.sum of ONE launch from `ncu --set "
               "full` (profiles/*_ncu_full_*.txt); compulsory attention bytes: Wan Q+K+V+O+LSE = "
               "404.2 MB, Cog 439.9 MB"}
    for wl, rep in (("wan", "full_wan.ncu-rep"), ("cog", "full_cog.ncu-rep")):
        p = os.path.join(SRC, rep)
        if not os.path.exists(p):
            continue
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), p],
                              capture_output=True, text=True).stdout
        open(os.path.join(DST, f"{tag}_ncu_full_{wl}.txt"), "w").write(summ)
        d = dram(p)
        traffic[wl] = {("attn" if k.startswith("attn") else k.replace("_kernel", "")): v
                       for k, v in d.items()}
    for wl in ("wan", "cog"):  # backward kernels (F3), not part of the bench roofline
        p = os.path.join(SRC, f"full_bwd_{wl}.ncu-rep")
        if os.path.exists(p):
            summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"),
                                   p], capture_output=True, text=True).stdout
            open(os.path.join(DST, f"{tag}_ncu_full_bwd_{wl}.txt"), "w").write(summ)
            traffic[f"bwd_{wl}"] = {k.replace("_kernel", ""): v for k, v in dram(p).items()}
    json.dump(traffic, open(os.path.join(DST, "traffic.json"), "w"), indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
