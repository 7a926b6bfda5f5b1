"""Summarise the ncu evidence of scripts/prof_round.sh (gpurun_out/) into profiles/ (committed):

* profiles/<tag>_launches_one_step.csv -- the launch list of one bench step;
* profiles/<tag>_ncu_step.md -- the full capture of the 13 tc_gemm launches of one step
  (tensor %, DRAM bytes, L2->SM TMA bytes, clocks) and the per-launch traffic the bench
  line's roofline.traffic reports (profiles/traffic.json);
* profiles/<tag>_ncu_algorithms.md -- one execute of VGG conv1_2 and conv3_2 for every
  algorithm: per kernel duration, tensor / FMA pipe %, DRAM GB/s and bytes, TMA bytes.

usage: python scripts/summarize_r02.py [tag]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.environ.get("PROF_OUT", os.path.join(ROOT, "profiles"))
RUN = os.environ.get("PROF_RUN", os.path.join(ROOT, "gpurun_out"))
os.makedirs(OUT, exist_ok=True)
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"

METRICS = {"gpu__time_duration.sum": "us", "sm__cycles_elapsed.avg.per_second": "sm_hz",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pct",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_cyc_pct",
           "dram__bytes_read.sum": "dram_rd", "dram__bytes_write.sum": "dram_wr",
           "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum": "tma_ld",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct"}
SCALE = {"s": 1e6, "ms": 1e3, "us": 1, "ns": 1e-3, "second": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def read_rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")[:48]}
        for k, name in METRICS.items():
            if k in h:
                i = h.index(k)
                try:
                    d[name] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    d[name] = float("nan")
        out.append(d)
    return out


def fmt(d, k, scale=1.0, nd=1):
    v = d.get(k)
    return "-" if v is None or v != v else f"{v * scale:.{nd}f}"


# ---- launch list of one bench step (the last 14 ai3 launches: conv1_1 prep + 13 GEMMs)
rows = [r for r in csv.reader(l for l in open(os.path.join(RUN, "launches.csv")) if not l.startswith("=="))]
h = rows[0]
launches = [(dict(zip(h, r))["ID"], dict(zip(h, r))["Kernel Name"].split("(")[0].replace("void ", ""),
             float(dict(zip(h, r))["Metric Value"])) for r in rows[1:]
            if dict(zip(h, r)).get("Metric Name") == "gpu__time_duration.sum" and "ai3::" in dict(zip(h, r))["Kernel Name"]]
step = launches[-14:]
with open(os.path.join(OUT, f"{tag}_launches_one_step.csv"), "w") as f:
    f.write("id,kernel,duration_ns\n")
    for i, k, t in step:
        f.write(f"{i},{k},{t:.0f}\n")
tot = sum(t for _, _, t in step)
tc = sum(t for _, k, t in step if "tc_gemm" in k)

# ---- full capture of the 13 tc_gemm launches of one step
names = ["conv1_1", "conv1_2", "conv2_1", "conv2_2", "conv3_1", "conv3_2", "conv3_3", "conv4_1", "conv4_2", "conv4_3",
         "conv5_1", "conv5_2", "conv5_3"]
kern = read_rep(os.path.join(RUN, "prof_step.ncu-rep"))
lines = [f"# ncu: one bench step ({tag})", "",
         "`scripts/prof_round.sh` on a B200 under gpurun: `bench.py --quick` step = the 13 VGG-16 convs, N=64, bf16,",
         "NHWC, `guess` (every layer on `implicit_gemm`).", "",
         "## Launch list (`--metrics gpu__time_duration.sum --clock-control none`; cold, serialised: compare shares)", "",
         f"Total {tot / 1e3:.1f} us; `tc_gemm_kernel` share {100 * tc / tot:.1f} %.", "",
         "| id | kernel | us |", "|---|---|---|"]
lines += [f"| {i} | {k} | {t / 1e3:.1f} |" for i, k, t in step]
lines += ["", "## Full capture (`--set full`) of the 13 `tc_gemm_kernel` launches", "",
          "ncu replays each launch ~40 times at its own clocks (SM GHz column), so durations differ from the bench's.", "",
          "| layer | us | SM GHz | tensor active % | DRAM rd MB | DRAM wr MB | DRAM % | L2->SM TMA GB | L2 % |",
          "|---|---|---|---|---|---|---|---|---|"]
traffic = []
for j, d in enumerate(kern):
    traffic.append(d.get("dram_rd", 0) + d.get("dram_wr", 0))
    lines.append(f"| {names[j] if j < len(names) else j} | {fmt(d, 'us')} | {fmt(d, 'sm_hz', 1e-9, 3)} | "
                 f"{fmt(d, 'tensor_pct')} | {fmt(d, 'dram_rd', 1e-6)} | {fmt(d, 'dram_wr', 1e-6)} | "
                 f"{fmt(d, 'dram_pct')} | {fmt(d, 'tma_ld', 1e-9, 2)} | {fmt(d, 'l2_pct')} |")
open(os.path.join(OUT, f"{tag}_ncu_step.md"), "w").write("\n".join(lines) + "\n")
if len(traffic) >= 12:
    tcl = traffic[1:13]  # the 12 tensor-bound layers (the roofline's dominant kernel), one launch each
    json.dump({"bytes_per_launch": sum(tcl) / len(tcl),
               "per_launch": {names[j + 1]: tcl[j] for j in range(len(tcl))},
               "note": f"mean dram__bytes_read.sum + dram__bytes_write.sum over the 12 tensor-bound tc_gemm_kernel "
                       f"launches (conv1_2 .. conv5_3) of one bench step ({tag}, profiles/{tag}_ncu_step.md)"},
              open(os.path.join(OUT, "traffic.json"), "w"), indent=1)

# ---- one execute per (layer, algorithm)
alines = [f"# ncu: one execute per algorithm ({tag})", "",
          "`scripts/prof_round.sh`: `scripts/prof_layer.py <layer> <algo>` (VGG-16, N=64, bf16, NHWC), one plan execute",
          "captured with `ncu --set full --profile-from-start off`.  Algorithmic bytes: conv1_2 822 MB, conv3_2 207 MB;",
          "FLOPs 236.8 G each (direct count).", "",
          "| layer | algorithm | kernel | us | tensor % | FMA % | DRAM rd MB | DRAM wr MB | DRAM GB/s | TMA ld GB | warps active % |",
          "|---|---|---|---|---|---|---|---|---|---|---|"]
for layer in ("conv1_2", "conv3_2"):
    for algo in ("implicit_gemm", "implicit_precomp_gemm", "winograd", "gemm", "kn2row", "direct", "smm"):
        p = os.path.join(RUN, f"prof_{layer}_{algo}.ncu-rep")
        if not os.path.exists(p):
            continue
        ks = read_rep(p)
        agg = {}
        for d in ks:  # kn2row: 9 tap GEMMs of one kernel -> aggregate per kernel name
            a = agg.setdefault(d["kernel"], {"n": 0, "us": 0.0, "dram_rd": 0.0, "dram_wr": 0.0, "tma_ld": 0.0,
                                              "tensor_pct": 0.0, "fma_pct": 0.0, "occ_pct": 0.0})
            a["n"] += 1
            for k in ("us", "dram_rd", "dram_wr", "tma_ld"):
                a[k] += d.get(k, 0.0) if d.get(k) == d.get(k) else 0.0
            for k in ("tensor_pct", "fma_pct", "occ_pct"):
                a[k] += (d.get(k, 0.0) if d.get(k) == d.get(k) else 0.0) * d.get("us", 0.0)
        for k, a in agg.items():
            us = a["us"]
            w = lambda name: a[name] / us if us else float("nan")  # noqa: E731
            alines.append(f"| {layer} | {algo} | {k}{' x' + str(a['n']) if a['n'] > 1 else ''} | {us:.1f} | "
                          f"{w('tensor_pct'):.1f} | {w('fma_pct'):.1f} | {a['dram_rd'] / 1e6:.1f} | {a['dram_wr'] / 1e6:.1f} | "
                          f"{(a['dram_rd'] + a['dram_wr']) / (us * 1e3) if us else 0:.0f} | {a['tma_ld'] / 1e9:.2f} | "
                          f"{w('occ_pct'):.1f} |")
open(os.path.join(OUT, f"{tag}_ncu_algorithms.md"), "w").write("\n".join(alines) + "\n")
print("\n".join(lines))
print()
print("\n".join(alines))
