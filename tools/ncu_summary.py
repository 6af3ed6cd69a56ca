"""Print key metrics of ncu --set full reports as a markdown table (one column per report), and
the per-launch DRAM bytes (for profiles/ncu_traffic.json)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "smsp__inst_executed.sum"]


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[-1]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    d["_kernel"] = (d.get("Kernel Name", ("?", ""))[0], "")
    return d


reps = sys.argv[1:]
ms = [metrics(r) for r in reps]
print("| metric | " + " | ".join(reps) + " |")
print("|---|" + "---|" * len(reps))
for k in ["_kernel"] + KEYS:
    print(f"| `{k}` | " + " | ".join(f"{m.get(k, ('-', ''))[0]} {m.get(k, ('', ''))[1]}".strip() for m in ms) + " |")
for r, m in zip(reps, ms):
    def val(key):
        x, unit = m[key]
        x = float(x.replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    print(f"{r}: dram bytes per launch = {val('dram__bytes_read.sum') + val('dram__bytes_write.sum'):.6e}")
