"""Summarise one round's ncu captures into profiles/ (tracked).

usage: python tools/profile_summary.py TAG [envs requests]

Reads gpurun_out/prof_rollout_TAG.ncu-rep, prof_reduce_TAG.ncu-rep and
launches_TAG.csv (written by tools/gpu_round.sh on the GPU box) and writes
  profiles/TAG_ncu_<kernel>.txt      key metrics + per-source-line hot spots
  profiles/TAG_launches.csv          the gpu__time_duration launch list
  profiles/ncu_summary.json          per-kernel DRAM traffic (read by bench.py)
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

KERNELS = {"rollout": ("rollout.o", "rollout_kernelILi3ELi16"), "reduce": ("reduce.o", "reduce_kernelILi5"),
           "route_tc": ("route_tc.o", "route_tc_kernelILi3ELi8")}


def metric(d, k):
    v = d.get(k)
    return None if v is None else float(v[0].replace(",", ""))


def main():
    tag = sys.argv[1]
    envs = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
    reqs = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
    out_dir = os.path.join(ROOT, "profiles")
    os.makedirs(out_dir, exist_ok=True)
    summ_path = os.path.join(out_dir, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {"kernels": {}}
    for name, (obj, ksub) in KERNELS.items():
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{name}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            continue
        # the report itself is kept beside its summary (tracked; .gpurunignore keeps it off the box)
        shutil.copyfile(rep, os.path.join(out_dir, f"{tag}_prof_{name}.ncu-rep"))
        d = ncu_summary.summary(rep)[0]
        unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        def nbytes(k):
            v = d.get(k)
            return None if v is None else float(v[0].replace(",", "")) * unit.get(v[1], 1.0)
        rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
        t_ms = metric(d, "gpu__time_duration.sum")
        if t_ms is not None and d["gpu__time_duration.sum"][1] == "us":
            t_ms *= 1e-3
        summ["kernels"][name] = dict(
            tag=tag, kernel=d["kernel"], envs=envs, requests=reqs, time_ms=t_ms,
            dram_read_bytes=rd, dram_write_bytes=wr, dram_bytes=(rd or 0) + (wr or 0),
            issue_active_pct=metric(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            dram_pct=metric(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            fp64_pipe_pct=metric(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            tensor_pipe_pct=metric(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
            warps_active=metric(d, "sm__warps_active.avg.per_cycle_active"),
            registers=metric(d, "launch__registers_per_thread"),
            source=f"ncu --set full --clock-control none, report profiles/{tag}_prof_{name}.ncu-rep")
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, v = rows[0], rows[2]
        for k in ("smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"):
            if k in h:
                summ["kernels"][name][k] = float(v[h.index(k)].replace(",", ""))
        lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep,
                                os.path.join(ROOT, "paper_2401_07886_b200", "csrc", "build", obj), ksub,
                                "40"], capture_output=True, text=True).stdout
        with open(os.path.join(out_dir, f"{tag}_ncu_{name}.txt"), "w") as f:
            f.write(f"# {d['kernel']}  ({envs} envs x {reqs} requests, tools/gpu_round.sh {tag})\n")
            for k, val in d.items():
                if k != "kernel":
                    f.write(f"{k:70s} {val}\n")
            f.write("\n# hot source lines (tools/ncu_lines.py): share of warp-stall samples and of "
                    "executed instructions\n")
            f.write(lines)
    # training-loop kernels (prof_train_TAG / prof_step_tc_TAG: several kernels per report):
    # per-launch DRAM bytes, time, HBM GB/s, issue and pipe activity (read by bench.py)
    for rep_name in ("train", "step_tc"):
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{rep_name}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            rep = os.path.join(out_dir, f"{tag}_prof_{rep_name}.ncu-rep")
        if not os.path.exists(rep):
            continue
        if rep_name == "train":
            summ["kernels"]["_train"] = {}  # this report replaces the previous training kernels
        for d in ncu_summary.summary(rep):
            kname = d["kernel"].split("(")[0].replace("void ", "").split("<")[0].strip()
            if kname in summ["kernels"].get("_train", {}):
                continue  # first launch of each kernel
            unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
            def nb(k, d=d):
                v = d.get(k)
                return None if v is None else float(v[0].replace(",", "")) * unit.get(v[1], 1.0)
            t = metric(d, "gpu__time_duration.sum")
            t_us = t * (1e3 if d["gpu__time_duration.sum"][1] == "ms" else 1.0)
            b = (nb("dram__bytes_read.sum") or 0) + (nb("dram__bytes_write.sum") or 0)
            summ["kernels"].setdefault("_train", {})[kname] = dict(
                tag=tag, time_us=t_us, dram_bytes=b, hbm_gbs=b / (t_us * 1e-6) / 1e9,
                issue_active_pct=metric(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                tensor_pipe_pct=metric(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                fp64_pipe_pct=metric(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                source=f"ncu --set full --clock-control none, report profiles/{tag}_prof_{rep_name}.ncu-rep "
                       "(config 3: 4,096 envs, batch 512)")
    launches = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if os.path.exists(launches):
        shutil.copy(launches, os.path.join(out_dir, f"{tag}_launches.csv"))
    json.dump(summ, open(summ_path, "w"), indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
