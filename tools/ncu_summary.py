"""Print the key ncu metrics of a .ncu-rep (raw page) — used to fill profiles/."""
import csv, subprocess, sys, json
WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.per_cycle_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__cycles_elapsed.avg.per_second',
        'lts__t_bytes.sum']
def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for w in WANT:
            if w in h:
                d[w] = (v[h.index(w)], u[h.index(w)])
        stalls = {h[i]: float(v[i].replace(",", "")) for i in range(len(h))
                  if h[i].startswith("smsp__average_warp_latency_issue_stalled") and h[i].endswith(".ratio") and v[i]}
        d["top_stalls"] = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        res.append(d)
    return res
if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in summary(p):
            print("==", p, d["kernel"][:60])
            for k, v in d.items():
                if k not in ("kernel",):
                    print(f"   {k:70s} {v}")
