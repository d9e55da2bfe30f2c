"""Summarise an ncu --set full report of the path's kernels (run here, no GPU):
per-kernel duration, DRAM bytes, DRAM/SM throughput and the top stall reasons.
Writes profiles/<name>_ncu.csv and profiles/<config>_traffic.json
(stage index -> dram read+write bytes per launch, read by bench.py)."""
import csv
import io
import json
import subprocess
import sys

rep, name, config = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
M = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
     "smsp__average_warp_latency_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_barrier"]
scale = {"ms": 1, "us": 1e-3, "ns": 1e-6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1, "second": 1e3}
out = []
stage_of = [("k1_", 0), ("k_fft_mid_tma<512, (int)-1", 1), ("k_fft_mid<", None), ("k3_", 2), ("k_fft_mid_tma<", 3), ("k4_", 4)]
traffic = {}
seen = 0
for r in rows[2:]:
    d = {}
    for m in M:
        if m in hdr:
            i = hdr.index(m)
            v = r[i]
            u = units[i]
            if u in scale:
                v = float(v.replace(",", "")) * scale[u]
            d[m] = v
    out.append(d)
with open(f"profiles/{name}_ncu.csv", "w", newline="") as fh:
    w = csv.DictWriter(fh, fieldnames=[m for m in M if m in hdr])
    w.writeheader()
    for d in out:
        w.writerow(d)
# kernel -> stage slot (K1 0, K2 1, K3 / fused pass B 2, K4a 3, K4b 4)
def slot(name):
    if "k1_" in name:
        return 0
    if "k_passb" in name or "k3_" in name:
        return 2
    if "k4_" in name:
        return 4
    if "k_fft_mid" in name:
        return 1 if ("(int)-1" in name or ", -1>" in name) else 3
    return None
for d in out:
    sl = slot(d["Kernel Name"])
    if sl is not None and str(sl) not in traffic:
        traffic[str(sl)] = int(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"])
json.dump(traffic, open(f"profiles/{config}_traffic.json", "w"))
for d in out:
    print(d["Kernel Name"][:50], "ms=%.4f" % d["gpu__time_duration.sum"], "R=%.3fGB W=%.3fGB" % (
        d["dram__bytes_read.sum"] / 1e9, d["dram__bytes_write.sum"] / 1e9),
        "dram%%=%s sm%%=%s regs=%s" % (d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                                      d.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                                      d.get("launch__registers_per_thread")))
