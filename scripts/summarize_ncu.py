"""Summarise gpurun_out/ ncu evidence into profiles/ (committed): launch list of one bench
step, per-kernel full-capture metrics, and the dominant kernel's DRAM traffic per launch."""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(OUT, exist_ok=True)

# ---- launch list: keep the last bench step (the kernels after the final warm-up step)
rows = [r for r in csv.reader(open(os.path.join(ROOT, "gpurun_out", "launches.csv"))) if len(r) > 10]
h = rows[0]
launches = []
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") == "gpu__time_duration.sum" and "ai3::" in d["Kernel Name"]:
        launches.append((d["ID"], d["Kernel Name"].split("(")[0].replace("void ", ""), float(d["Metric Value"])))
per_step = 14  # conv1_1: prep + tc; 12 more tc launches
step = launches[-per_step:]
with open(os.path.join(OUT, f"{tag}_launches_one_step.csv"), "w") as f:
    f.write("id,kernel,duration_ns\n")
    for i, k, t in step:
        f.write(f"{i},{k},{t:.0f}\n")
tot = sum(t for _, _, t in step)
tc = sum(t for _, k, t in step if "tc_gemm" in k)

# ---- full capture metrics
rep = os.path.join(ROOT, "gpurun_out", "prof_step.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh, units = rr[0], rr[1]
want = {"gpu__time_duration.sum": "duration", "sm__cycles_elapsed.avg.per_second": "sm_clock",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_active_pct",
        "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum": "tma_load_bytes",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
        "launch__grid_size": "grid", "launch__registers_per_thread": "regs"}
kern = []
for r in rr[2:]:
    d = {}
    for k, name in want.items():
        if k in hh:
            d[name] = (r[hh.index(k)], units[hh.index(k)])
    kern.append(d)

def to_bytes(v, u):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return float(v) * mult.get(u, 1)

lines = [f"# ncu summary ({tag})", "",
         "Source: `scripts/profile_round.sh` on a B200 (gpurun), `bench.py` step = the 13 VGG-16 convs, N=64, bf16, NHWC, `guess`.",
         "", "## Launch list of one step (cold-cache, serialised: compare shares, not absolutes)", "",
         f"Total {tot/1e3:.1f} us; tc_gemm_kernel share {100*tc/tot:.1f}%.", "", "| id | kernel | us |", "|---|---|---|"]
lines += [f"| {i} | {k} | {t/1e3:.1f} |" for i, k, t in step]
lines += ["", "## Full capture (`ncu --set full`) of tc_gemm_kernel launches", "",
          "| # | us | SM GHz | tensor active % | DRAM read MB | DRAM write MB | TMA load GB | L2 % | DRAM % |",
          "|---|---|---|---|---|---|---|---|---|"]
traffic = []
for j, d in enumerate(kern):
    g = lambda n: d.get(n, ("nan", ""))
    rd = to_bytes(*g("dram_read")); wr = to_bytes(*g("dram_write"))
    traffic.append(rd + wr)
    lines.append(f"| {j} | {float(g('duration')[0]):.1f} | {float(g('sm_clock')[0]):.3f} | {float(g('tensor_active_pct')[0]):.1f} | "
                 f"{rd/1e6:.1f} | {wr/1e6:.1f} | {to_bytes(*g('tma_load_bytes'))/1e9:.2f} | {float(g('l2_throughput_pct')[0]):.1f} | "
                 f"{float(g('dram_throughput_pct')[0]):.1f} |")
open(os.path.join(OUT, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
if traffic:
    json.dump({"bytes_per_launch": sum(traffic) / len(traffic),
               "note": f"mean dram__bytes_read.sum + dram__bytes_write.sum over {len(traffic)} captured tc_gemm_kernel "
                       f"launches of the bench step ({tag}, profiles/{tag}_ncu_summary.md)"},
              open(os.path.join(OUT, "traffic.json"), "w"), indent=1)
print("\n".join(lines))
