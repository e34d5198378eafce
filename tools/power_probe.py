"""Dev tool: steady-state time, SM clock and board power of one config run back to back.

Runs the C-ABI call of a bench config for --seconds after a warm-up, sampling NVML every 20 ms,
and prints one JSON line: ms per call, per-class kernel times (library events, second pass),
median SM clock, median / max board power.  Used to attribute power under sw_power_cap to the
parts of the leaf (ADJ_LEAF_DEBUG diagnostic switches change the work, not the result check).
"""
import argparse
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2101_01025_b200 as adj  # noqa: E402
from bench import CONFIGS  # noqa: E402
from inputs.gpu import uniform_residues_cuda  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--depth", type=int, default=None)
ap.add_argument("--seconds", type=float, default=4.0)
ap.add_argument("--flags", type=int, default=-1, help="adjprod flags (default: uint16 I/O when p < 2^16)")
ap.add_argument("--tag", default="")
ap.add_argument("--lowmem", action="store_true", help="ADJ_LOW_MEM schedule")
a = ap.parse_args()
cfg = CONFIGS[a.config]
m, k, p = cfg["m"], cfg["k"], cfg["p"]
w = 2 if cfg["phi"] == "H" else 1
phi = 1 if w == 2 else 0
io16 = p < 65536 and a.flags < 0
A = torch.empty((m, k * w), dtype=torch.int32, device="cuda")
uniform_residues_cuda(A, 1, p)
C = torch.zeros((m, m * w), dtype=torch.int32, device="cuda")
flags = max(a.flags, 0)
if io16:
    A, C = A.to(torch.int16), C.to(torch.int16)
    flags = adj.ADJ_IN_U16 | adj.ADJ_OUT_U16
if a.lowmem:
    flags |= adj.ADJ_LOW_MEM
d = a.depth if a.depth is not None else adj.adjprod_modp_auto_depth(m, k, p, phi)
wsb = adj.adjprod_modp_workspace_size(m, k, p, phi, d, flags=flags)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()


def call():
    adj.adjprod_modp_ex(m, k, p, phi, A, k, C, m, depth=d, flags=flags, workspace=ws, workspace_bytes=wsb, stream=s)


for _ in range(3):
    call()
torch.cuda.synchronize()

import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.02)


th = threading.Thread(target=sampler)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
th.start()
n = 0
t0 = time.time()
e0.record(s)
while time.time() - t0 < a.seconds:
    call()
    n += 1
    if n % 4 == 0:
        torch.cuda.synchronize()
e1.record(s)
torch.cuda.synchronize()
stop.set()
th.join()
ms = e0.elapsed_time(e1) / n
adj.adj_profile_enable(True)
adj.adj_profile_read()
for _ in range(3):
    call()
torch.cuda.synchronize()
prof = adj.adj_profile_read()
adj.adj_profile_enable(False)
half = samples[len(samples) // 4:]
mhz = sorted(x[0] for x in half)
pw = sorted(x[1] for x in half)
print(json.dumps({"tag": a.tag, "config": a.config, "depth": d, "leaf_debug": os.environ.get("ADJ_LEAF_DEBUG", "0"),
                  "calls": n, "ms_per_call": round(ms, 4),
                  "classes_ms": {c: round(v[0] / 3, 4) for c, v in prof.items()},
                  "sm_mhz_median": mhz[len(mhz) // 2] if mhz else None,
                  "power_w_median": round(pw[len(pw) // 2], 1) if pw else None,
                  "power_w_max": round(pw[-1], 1) if pw else None, "workspace_bytes": wsb}))
