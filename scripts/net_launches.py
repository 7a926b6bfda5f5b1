"""One pass over a network's unique conv layers (BASELINE configs, `guess`), for an ncu launch
list: python scripts/net_launches.py resnet50 256  (run under ncu --metrics gpu__time_duration.sum).
With --summarize CSV it writes the per-layer kernel table (markdown) to stdout instead."""
import csv, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if sys.argv[1] == "--summarize":
    rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ks = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi]) / 1e3) for r in rows[1:] if "ai3::" in r[ki]]
    names = [l.strip() for l in open(sys.argv[3])]
    # the script's last pass: the last sum(launches per layer) ai3 launches
    ks = ks[-sum(int(n.split()[1]) for n in names):]
    print("| layer | kernels (us) | total us |\n|---|---|---|")
    i = 0
    for name in names:
        lay, n = name.split()
        n = int(n)
        part = ks[i:i + n]
        i += n
        print(f"| {lay} | " + ", ".join(f"{k.replace('ai3::', '')} {t:.1f}" for k, t in part) +
              f" | {sum(t for _, t in part):.1f} |")
    sys.exit(0)

import torch
import paper_2410_08300_b200 as ai3
from synth import workload, conv_inputs
net, batch = sys.argv[1], int(sys.argv[2])
plans = []
for l in workload(net, batch):
    x = torch.randn(l.N, l.C, l.H, l.W, device="cuda").bfloat16().contiguous(memory_format=torch.channels_last)
    _, w, b = conv_inputs(l.with_batch(1), 1, "bf16")
    p = ai3.ConvPlan(torch.from_numpy(w).cuda().bfloat16(), None if b is None else torch.from_numpy(b).cuda().bfloat16(),
                     x.shape, l.stride, l.pad, l.dil, 1, "guess", in_layout=1)
    plans.append((l.name, p, x, p(x)))
with open(os.path.join(ROOT, "gpurun_out", f"{net}_layers.txt"), "w") as f:
    for name, p, _, _ in plans:
        f.write(f"{name} {p.num_launches}\n")
for _ in range(2):  # pass 1 warm-up, pass 2 is the one summarised
    for name, p, x, y in plans:
        p(x, out=y)
torch.cuda.synchronize()
