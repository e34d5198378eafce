"""Dev tool: print step / kernel times of gpurun_out/ab_*.json."""
import glob
import json

for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    hk = d.get("hbm_kernels") or {}
    print(f, f"step {d['ms_per_step']:.4f} ms leaf {d['roofline']['leaf_ms_per_launch']:.4f} frac {d['roofline']['frac']:.3f}",
          " ".join(f"{k} {v['ms']:.4f} ({v['frac']:.2f})" for k, v in hk.items()))
