"""Print DESIGN.md §9's measured table rows from profiles/<tag>_bench_*.jsonl (one line per config)."""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02f"
names = {"small": "small (d = 1000, k = 10)", "medium": "medium (d = 256, k = 20)",
         "large": "**large** (bench default)", "xl": "xl on one GPU (k = 100)"}
for c in ["small", "medium", "large", "xl"]:
    d = json.loads(open(f"profiles/{tag}_bench_{c}.jsonl").readline())
    st = d["stages_ms"]
    e2e = d.get("e2e") or {}
    cb = d.get("cpu_baseline") or {}
    step = f"**{d['ms_per_step']:.1f}**" if c == "large" else (f"{d['ms_per_step']:.0f}" if c == "xl" else f"{d['ms_per_step']:.1f}")
    row = [names[c], step, f"{st['propagate']:.1f}", f"{st['features']:.1f}", f"{st['topk_eig']:.1f}", f"{st['cluster']:.1f}",
           f"{e2e['ms_per_step']:.1f}" if e2e.get("ms_per_step") else "—",
           f"{d['propagation_nnz_d_per_s'] / 1e12:.2f} T", f"{d['roofline']['frac']:.3f}",
           f"{cb['tpo_seconds']:.1f}" if cb.get("tpo_seconds") else "—"]
    print("| " + " | ".join(row) + " |")
