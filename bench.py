#!/usr/bin/env python
"""Benchmark of the hot path C = Low(A phi(A)) mod p (BASELINE.json metric: effective m^2 k
modular MAC/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--depth D] [--impl reference]

Default workload: c3 = BASELINE.json configs[2] (A 32768 x 32768 over GF(65521)), the config the
metric is quoted on at 1/2/4/8 B200.  One step = one adjprod_modp call (every §8(a) row:
pre-additions, grouped tcgen05 leaves, recombination, 2M combine for phi = H) on a seeded
uniform-residue A already resident in HBM.  L2 is flushed (256 MiB write) before every timed
step, outside the step's CUDA events.  Rank 0 prints ONE JSON line.  N > 1 (torchrun, or
`--gpus N` alone, which starts N ranks itself): adjprod_modp_dist over NCCL, strong scaling,
time = max over ranks.  --impl reference times the CPU oracle (oracle/) on host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(m=256, k=256, p=97, phi="T", depth=1,
               workload="c1: A 256x256 over GF(97), C = Low(A A^T) mod 97, Y = 22 I, one recursion level"),
    # c2 runs at the library's automatic depth, 0 at this size (classical is 5-8% faster on B200:
    # K1 + K4 cost more than the 1/8 of the MMAs one level saves on an L2-bound leaf); one level
    # of Alg. 1 is reported beside it (comparators.depth1_alg1)
    "c2": dict(m=8192, k=8192, p=8191, phi="T", depth=None,
               workload="c2: A 8192x8192 over GF(8191), C = Low(A A^T) mod 8191, Y = Rot2(2670, 5929)"),
    "c3": dict(m=32768, k=32768, p=65521, phi="T", depth=None,
               workload="c3: A 32768x32768 over GF(65521), C = Low(A A^T) mod 65521, Y = 24297 I"),
    "c4": dict(m=16384, k=131072, p=8191, phi="T", depth=None,
               workload="c4: A 16384x131072 over GF(8191), C = Low(A A^T) mod 8191 (16384^2)"),
    "x16k": dict(m=16384, k=16384, p=8191, phi="T", depth=None,
                 workload="x16k (dev): A 16384x16384 over GF(8191)"),
    "x131071": dict(m=8192, k=8192, p=131071, phi="T", depth=None,
                    workload="x131071 (dev): A 8192x8192 over GF(131071), the paper's modulus (PAPER.md:2237)"),
    "x131071_32k": dict(m=32768, k=32768, p=131071, phi="T", depth=None,
                        workload="x131071_32k (dev): A 32768x32768 over GF(131071), the paper's modulus at c3 size"),
    "x65521": dict(m=8192, k=8192, p=65521, phi="T", depth=None,
                   workload="x65521 (dev): A 8192x8192 over GF(65521)"),
    "x251": dict(m=8192, k=8192, p=251, phi="T", depth=None,
                 workload="x251 (dev): A 8192x8192 over GF(251), one int8 limb"),
    "c5": dict(m=8192, k=8192, p=8191, phi="H", depth=None,
               workload="c5: A 8192x8192 over GF(8191^2) = GF(8191)[i]/(i^2+1), C = Low(A A^H) via 2M"),
    "q5": dict(m=8192, k=8192, p=8191, phi="Q", depth=None,
               workload="q5 (SURVEY 8(f)-4): M 8192x8192 over the quaternions H_GF(8191), C = Low(M M^H) via "
                        "Alg. 2M3M (6M)"),
}
# N = 1 headline: BASELINE.json configs[2] (c3), the configuration its metric is quoted on at
# 1/2/4/8 B200 (c4 is the other one; c1, c2, c5 are parity cases and --config options)
DEFAULT_CONFIG = "c3"
BASELINE_INDEX = {"c1": 0, "c2": 1, "c3": 2, "c4": 3, "c5": 4}
UNIT = "MAC/s"


def metric_label(name: str) -> str:
    """BASELINE.json's metric, labelled with the config it is measured on."""
    where = (f"BASELINE configs[{BASELINE_INDEX[name]}]" if name in BASELINE_INDEX
             else "SURVEY 8(f) / dev config")
    return f"effective m^2 k modular MAC/s for C=A*A^T mod p at N B200 ({name}: {where})"


def config_dict(name: str, cfg) -> dict:
    """The workload, identical on both arms (--impl ours / reference): what is computed, not how."""
    return {"workload": cfg["workload"], "id": name, "m": cfg["m"], "k": cfg["k"], "p": cfg["p"], "phi": cfg["phi"],
            "seed": 1, "inputs": "uniform residues in [0, p) (inputs/: splitmix64 counter generator)",
            "l2": "inputs larger than L2 and a 256 MiB L2 flush before every timed step (outside step events)"}


def limb_mmas(p: int) -> int:
    """int8 tcgen05 MMAs per ring MAC of the limb scheme."""
    return 1 if p <= 255 else (3 if p <= 16763 else (4 if p <= 65521 else 6))


def ring_macs(m: int, k: int, d: int) -> float:
    """Ring MACs the method performs: R_0 = m(m+1)/2 k (lower-triangle SYRK),
    R_d = 3 R_{d-1}(m/2, k/2) + 2 (m/2)^2 (k/2)  (Alg. alg:MIAHMM)."""
    if d == 0:
        return m * (m + 1) / 2 * k
    mh, kh = -(-m // 2), -(-k // 2)
    return 3 * ring_macs(mh, kh, d - 1) + 2 * mh * mh * kh


def herk_alg1_macs(m: int, k: int) -> float:
    """Base-field MACs of one level of Alg. alg:MIAHMM over GF(p^2) (ADJ_HERK_ALG1): three
    Hermitian leaves by 2M (G = T T^T lower + H = X Y^T) and two general leaves by 3M."""
    mh, kh = -(-m // 2), 8 * -(-k // 16)
    return 3 * (mh * (mh + 1) / 2 * kh) + 9 * mh * mh * kh


def leaf_int8_ops(cfg, depth, herk="2m") -> float:
    """Algorithmic int8 tensor ops (2 per MAC) of ONE grouped leaf launch."""
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    if cfg["phi"] == "H" and herk == "alg1":
        return 2.0 * herk_alg1_macs(m, k) * limb_mmas(p)
    macs = ring_macs(m, k, depth)
    if cfg["phi"] == "H":
        macs += m * m * k            # 2M's general product H = X Y^T
    if cfg["phi"] == "Q":
        macs += 5 * m * m * k        # 6M's general products Q1..Q5 (Q6 is the ring_macs term)
    return 2.0 * macs * limb_mmas(p)


def k1_fused(cfg, depth, res_bytes):
    """the library's fused K1 of levels 1 + 2 runs (api.cpp k1_fused_ok): phi = T, depth >= 2,
    uint16 residues, m and k multiples of 512"""
    return (cfg["phi"] == "T" and depth >= 2 and res_bytes == 2 and cfg["p"] < 65536
            and cfg["m"] % 512 == 0 and cfg["k"] % 512 == 0)


def hbm_bytes(cfg, depth, herk="2m", res_bytes=4):
    """Algorithmic HBM bytes per step of the HBM-bound classes (K1 pre-addition / split and the
    recombination K4 / 2M / 6M combine), for the layouts DESIGN.md §4 describes: read each input
    once, write each limb plane (padded arena rows) / residue once.  Any depth for phi = T; depth 0
    for phi = H / Q; None for phi = H via ADJ_HERK_ALG1.
    res_bytes: bytes per caller residue of A and Low(C) (4, or 2 with ADJ_IN_U16 | ADJ_OUT_U16)."""
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    w = {"T": 1, "H": 2, "Q": 4}[cfg["phi"]]
    planes = {1: 1, 3: 3, 4: 2, 6: 6}[limb_mmas(p)]
    rp = lambda x: -(-x // 128) * 128
    res = 4 if p > 65535 else 2                             # workspace residues (S3, P buffers)
    out_c = m * (m + 1) // 2 * res_bytes * w                # Low(C), uint32 (or uint16) words
    if cfg["phi"] == "H" and herk == "alg1":
        return None
    if depth == 0:
        nops = {1: 1, 2: 3, 4: 7}[w]                       # A | X, Y, T | A, B, C, D, U1, U2, W
        pre = res_bytes * w * m * k + nops * planes * rp(m) * max(128, rp(k))
        if w == 1:
            comb = None                                    # the leaf epilogue writes C directly
        else:
            nbuf = {2: (1, 1), 4: (5, 1)}[w]               # full buffers read (H | Q1..Q5), lower ones (G | Q6)
            comb = (nbuf[0] * m * m + nbuf[1] * m * (m + 1) // 2) * res + out_c
        return {"preadd": pre, "combine": comb}
    if w != 1:
        return None
    # phi = T, depth >= 1: walk the recursion tree (api.cpp run_tree / run_combine).  Level l has
    # 3^(l-1) nodes of half sizes mh_l = ceil(mh_{l-1} / 2), kh_l = 8 ceil(kh_{l-1} / 16); K1 of a
    # node reads the valid part of its input (A's elements at the root and in the X11 / X12 views,
    # workspace residues in S3) and writes n_ops limb operands of planes x rows_pad x kpad bytes
    # (4 operands S1, S2, S4, X22 above the last level, 7 at it) plus its S3 residues above the
    # last level; K4 of a node reads P1, P2, P5 (lower) and P3, P4 (full) and writes Low of its
    # output (Low(C) at the root, the parent's P slot below it).
    mh, kh = [m], [k]
    for _ in range(depth):
        mh.append(-(-mh[-1] // 2))
        kh.append(8 * -(-kh[-1] // 16))
    pre = comb = 0
    fused = k1_fused(cfg, depth, res_bytes)   # levels 1 + 2 in one pass: A read once, level-1 S3 in registers

    def node(level, rows, cols, esz):
        nonlocal pre, comb
        pre_read = 0 if (fused and level == 2) else rows * cols * esz   # (level 3 reads as before)
        nops = 7 if level == depth else 4
        pre_write = nops * planes * rp(mh[level]) * max(128, rp(kh[level]))
        if level < depth and not (fused and level == 1 and depth == 2):
            pre_write += mh[level] * kh[level] * res       # S3, the third child's input
        pre += pre_read + pre_write
        m_l = mh[level]
        comb += (3 * m_l * (m_l + 1) // 2 + 2 * m_l * m_l) * res
        comb += out_c if level == 1 else mh[level - 1] * (mh[level - 1] + 1) // 2 * res
        if level < depth:
            node(level + 1, min(rows, m_l), min(cols, kh[level]), esz)                        # X11
            node(level + 1, min(rows, m_l), max(0, min(cols - kh[level], kh[level])), esz)   # X12
            node(level + 1, m_l, kh[level], res)                                            # S3
    node(1, m, k, res_bytes)
    return {"preadd": pre, "combine": comb}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


_CUDART = None


def memcpy2d_d2h(dst, dpitch, src, spitch, width, height, stream):
    """cudaMemcpy2DAsync device -> pinned host (one call per row block; not a batched copy)."""
    global _CUDART
    import ctypes
    if _CUDART is None:
        _CUDART = ctypes.CDLL("libcudart.so.12")
        _CUDART.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                              ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        _CUDART.cudaMemcpy2DAsync.restype = ctypes.c_int
    rc = _CUDART.cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, 2, stream)
    if rc != 0:
        raise RuntimeError(f"cudaMemcpy2DAsync failed: {rc}")


class ClockSampler:
    """Polls NVML (SM clock, max clock, throttle reasons) while the timed region runs."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev_index: int, period_s: float = float(os.environ.get("ADJ_CLOCK_PERIOD_S", "0.002"))):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.power = []
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w_max": max(self.power) if getattr(self, "power", None) else None}


def load_traffic(config: str, depth: int):
    """dram__bytes_read + dram__bytes_write per leaf launch from the committed ncu --set full
    summary (profiles/leaf_traffic.json) when it was captured for this config and depth."""
    path = os.path.join(ROOT, "profiles", "leaf_traffic.json")
    try:
        with open(path) as f:
            d = (json.load(f).get(config) or {}).get(str(depth))
        return d["dram_bytes_per_launch"] if d else None
    except Exception:
        return None


def load_pure_mma_sustained():
    """The pure tcgen05 kind::i8 rate with random operands back to back at the board's power cap
    (tools/mma_peak.cu sustain, profiles/r02/int8_mma_sustained.json): the tensor datapath's own
    ceiling under the cap, context beside the contract's 2 x bf16 sustained peak."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "int8_mma_sustained.json")) as f:
            return float(json.load(f)["sustained_random_operands"]["steady_median_tops"])
    except Exception:
        return None


# ------------------------------------------------------------------------------ oracle
def cpu_model() -> str:
    """the host CPU's model name (/proc/cpuinfo), for the cpu_baseline context"""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(cfg, A_host, budget_s: float):
    """Time the oracle (as it stands) on a slab of the last rows of Low(C) -- the longest rows --
    sized to ~budget_s of CPU work; returns (effective m^2 k MAC/s extrapolated, seconds, cores, desc)."""
    import numpy as np
    import oracle
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    H = cfg["phi"] == "H"
    f = {"T": oracle.syrk_t, "H": oracle.syrk_h, "Q": oracle.syrk_q}[cfg["phi"]]
    cores = oracle.num_threads()
    # calibration on a tiny slab
    r = max(1, min(m, 2))
    t0 = time.perf_counter()
    f(A_host, p, rows=(m - r, m))
    t_cal = time.perf_counter() - t0
    macs_cal = sum(i + 1 for i in range(m - r, m)) * k
    rate = macs_cal / max(t_cal, 1e-6)

    def rows_for(target):
        rows, macs = 1, 0
        while rows < m and macs < target:
            macs += (m - rows + 1) * k
            rows += 1
        return max(1, rows - 1)

    # a tiny slab underestimates the multi-threaded rate: re-size until the slab takes at least
    # half the budget (or covers the whole triangle)
    rows = rows_for(budget_s * rate)
    for _ in range(4):
        t0 = time.perf_counter()
        f(A_host, p, rows=(m - rows, m))
        t = time.perf_counter() - t0
        sample_macs = sum(i + 1 for i in range(m - rows, m)) * k
        if t >= 0.5 * budget_s or rows >= m:
            break
        rows = rows_for(budget_s * sample_macs / max(t, 1e-6))
    full_lower = m * (m + 1) / 2 * k
    t_full = t * full_lower / sample_macs
    eff = m * m * k / t_full
    field = {"T": "GF(p)", "H": "GF(p^2) hermitian", "Q": "quaternion H_GF(p) hermitian"}[cfg["phi"]]
    desc = (f"O1 oracle ({field} u64 triple loop, OpenMP) on rows "
            f"[{m - rows}, {m}) of Low(C) = {sample_macs:.3e} of {full_lower:.3e} lower-triangle MACs in {t:.2f} s; "
            f"value extrapolated to the full problem by MAC count ({t_full:.1f} s)")
    return eff, t, cores, desc, t_full


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle as it stands, on host cores, rank 0 only.  One step = the
    oracle on one bounded slab of the workload (the last rows of Low(C), the longest ones), sized
    to ~ADJ_REF_STEP_S seconds; ms_per_step is that measured slab time, value its effective
    m^2 k MAC/s (slab ring MACs scaled by m^2 k / full lower-triangle MACs)."""
    from inputs import uniform_matrix, uniform_matrix_ext, uniform_matrix_quat
    if rank != 0:
        return
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    A = {"T": uniform_matrix, "H": uniform_matrix_ext, "Q": uniform_matrix_quat}[cfg["phi"]](m, k, 1, p)
    per_step = float(os.environ.get("ADJ_REF_STEP_S", "2.0"))
    for _ in range(args.warmup):
        oracle_sample(cfg, A, per_step / 4)
    vals, secs, tfull = [], [], []
    cores, desc = None, None
    for _ in range(args.steps):
        eff, t, cores, desc, t_full = oracle_sample(cfg, A, per_step)
        vals.append(eff)
        secs.append(t)
        tfull.append(t_full)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": metric_label(args.config), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
        "ms_per_step_is": "measured: the oracle on one bounded slab of the workload per step (see cpu_baseline.sample)",
        "extrapolated_full_problem_ms": 1e3 * statistics.median(tfull),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "uint64", "data": "synthetic",
        "config": config_dict(args.config, cfg),
        "parallelism": f"CPU oracle, {cores} host threads (OpenMP)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def run_gpu(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2101_01025_b200 as adj
    from inputs.gpu import uniform_residues_cuda

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    m, k, p = cfg["m"], cfg["k"], cfg["p"]
    phi = {"T": adj.ADJ_PHI_T, "H": adj.ADJ_PHI_H, "Q": adj.ADJ_PHI_Q}[cfg["phi"]]
    w = {"T": 1, "H": 2, "Q": 4}[cfg["phi"]]
    alg1 = cfg["phi"] == "H" and args.herk == "alg1"
    flags = adj.ADJ_HERK_ALG1 if alg1 else 0
    depth = args.depth if args.depth is not None else (cfg["depth"] if cfg["depth"] is not None
                                                       else (1 if alg1 else adj.adjprod_modp_auto_depth(m, k, p, phi)))
    # N > 1: output-tile sharding for square phi = T problems (depth <= 1) with each rank's final
    # kernel storing its regions straight into rank 0's C over NVLink, split-K otherwise
    dist_mode = args.dist if args.dist != "auto" else ("tiles-p2p" if cfg["phi"] == "T" and k <= 2 * m else "splitk")
    dist_flags = 0
    if world > 1 and dist_mode == "tiles":
        dist_flags = adj.ADJ_DIST_TILES
    elif world > 1 and dist_mode == "tiles-p2p":
        dist_flags = adj.ADJ_DIST_TILES | adj.ADJ_DIST_P2P
    elif world > 1 and dist_mode == "p2p":
        dist_flags = adj.ADJ_DIST_P2P
    if dist_flags:
        depth = min(depth, 1)
    # residues of A and Low(C) live in HBM as uint16 when phi = T and p < 2^16 (ADJ_IN_U16 |
    # ADJ_OUT_U16; exact, the same arithmetic), else uint32.  --io u32 forces uint32.
    # (N > 1: uint16 A, uint32 Low(C) on the root -- the distributed entry point reads ADJ_IN_U16)
    # phi = H: (re, im) uint16 pairs; Alg. 1 over GF(p^2) reads them but writes uint32 (and the
    # distributed path takes phi = T only), so those runs keep uint32 residues throughout
    io16 = ((cfg["phi"] == "T" or (cfg["phi"] in ("H", "Q") and not alg1 and world == 1)) and p < 65536
            and args.io in ("auto", "u16"))
    if io16 and world == 1:
        flags |= adj.ADJ_IN_U16 | adj.ADJ_OUT_U16
    elif io16:
        dist_flags |= adj.ADJ_IN_U16
    A32 = torch.empty((m, k * w), dtype=torch.int32, device=dev)
    uniform_residues_cuda(A32, seed=1, p=p)
    A = A32.to(torch.int16) if io16 else A32
    del A32
    A_bytes = A.numel() * A.element_size()
    C = torch.zeros((m, m * w), dtype=torch.int16 if io16 and world == 1 else torch.int32, device=dev)

    def u32(t):
        """the residues of a device tensor as an int32 tensor (uint16 storage zero-extended)"""
        return (t.to(torch.int32) & 0xFFFF) if t.element_size() == 2 else t
    comm = None
    if world > 1:
        uid = adj.adj_comm_get_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        comm = adj.adj_comm_init(world, obj[0], rank)
        k0, k1 = adj.adj_dist_kslice(k, world, rank)
        ws_bytes = 0   # the library allocates stream-ordered workspace inside adjprod_modp_dist
    else:
        ws_bytes = adj.adjprod_modp_workspace_size(m, k, p, phi, depth, flags)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        if comm is None:
            adj.adjprod_modp_ex(m, k, p, phi, A, k, C, m, depth=depth, flags=flags, workspace=ws,
                                workspace_bytes=ws_bytes, stream=stream)
        else:
            adj.adjprod_modp_dist(m, k, p, phi, A, k, C, m, 0, comm, depth=depth, flags=dist_flags, stream=stream)

    dist_fallback = None
    if comm is not None and dist_mode == "tiles-p2p":
        # the fused mode needs the root's C exportable over CUDA IPC; every rank agrees on the
        # status inside the call, so all of them fall back together to the NCCL gather
        try:
            step()
            torch.cuda.synchronize()
        except adj.AdjError as e:
            dist_fallback = f"tiles-p2p unavailable ({e}); NCCL gather of result tiles"
            dist_mode, dist_flags = "tiles", (dist_flags & ~adj.ADJ_DIST_P2P)
    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()

    # ---------------- timed region: device time per step, L2 flushed before each step.  The
    # library's per-kernel events (adj_profile_*) cost ~3% of a c2 step, so the headline pass runs
    # without them; a second pass of the same K steps (same flushes) records them for the roofline
    # of the leaf kernel and the HBM fractions.
    def timed_pass(profile):
        adj.adj_launch_count_reset()
        adj.adj_profile_enable(profile)
        adj.adj_profile_read()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local_rank) as clk:
            for i in range(args.steps):
                flush.zero_()
                evs[i][0].record(stream)
                step()
                evs[i][1].record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches = adj.adj_launch_count()
        prof = adj.adj_profile_read()
        adj.adj_profile_enable(False)
        step_ms = [a.elapsed_time(b) for a, b in evs]
        ms = sum(step_ms) / len(step_ms)
        stats = {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)}
        if world > 1:
            t = torch.tensor([ms, stats["min"], stats["median"], stats["max"]], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t[0].item())
            stats = {"min": float(t[1].item()), "median": float(t[2].item()), "max": float(t[3].item())}
        timed_pass.stats = stats
        return ms, launches, prof, clk

    t_pass = time.perf_counter()
    ms, launches, _, clk = timed_pass(False)
    step_stats = timed_pass.stats   # of the headline pass (max over ranks)
    # an idle gap of ~3x the pass lets the board's power average recover, so that the profiled
    # pass runs under the same clocks as the headline one
    time.sleep(min(3.0, max(0.3, 3.0 * (time.perf_counter() - t_pass))))
    ms_prof, _, prof, clk_prof = timed_pass(True)
    value = m * m * k / (ms * 1e-3)
    # N > 1: each rank runs its share of the step's leaf work (and K1 / K4 bytes); the roofline and
    # the HBM fractions below divide the whole step's algorithmic work by the per-class device time
    # summed over the ranks (the per-GPU average), not by rank 0's share alone
    prof_all = prof
    if world > 1:
        cls = sorted(prof)
        t = torch.tensor([prof[c][0] for c in cls], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        prof_all = {c: (float(t[i].item()) / world, prof[c][1]) for i, c in enumerate(cls)}

    # ---------------- sustained: the same steps back to back for ~--sustain-s seconds (the board
    # reaches its power cap on long streams; context for the burst-regime headline above, and the
    # leaf fraction against the sustained peak)
    sustained = None
    if world == 1 and args.sustain_s > 0:
        n_sus = max(args.steps, int(args.sustain_s / max(ms * 1e-3, 1e-6)))
        adj.adj_profile_enable(True)
        adj.adj_profile_read()
        a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with ClockSampler(local_rank) as clk_s:
            a0.record(stream)
            for _ in range(n_sus):
                flush.zero_()
                step()
            b0.record(stream)
            torch.cuda.synchronize()
        prof_s = adj.adj_profile_read()
        adj.adj_profile_enable(False)
        ms_s = a0.elapsed_time(b0) / n_sus      # includes the L2 flush between steps
        peaks_s, _ = load_peaks()
        leaf_ms_s = prof_s["leaf"][0] / n_sus
        tops_s = leaf_int8_ops(cfg, depth, args.herk) / (leaf_ms_s * 1e-3) / 1e12
        sus_peak = 2.0 * peaks_s.get("bf16_tflops_sustained", peaks_s["bf16_tflops"])
        sustained = {"steps": n_sus, "ms_per_step_incl_flush": ms_s, "leaf_ms_per_launch": leaf_ms_s,
                     "leaf_achieved_tops": tops_s, "leaf_frac_of_sustained_peak": tops_s / sus_peak,
                     "sustained_peak_tops": sus_peak, "clocks": clk_s.summary()}

    # ---------------- end to end through the C ABI with host buffers (pinned), copies timed.
    # A stream of problems: step i copies its A (H2D), runs the C-ABI call, and reads back its
    # Low(C) row blocks (D2H); three streams, three A buffers and two C buffers, so step i's H2D
    # overlaps step i-1's compute and step i-2's D2H and may start one compute early (at c3 the
    # H2D of the uint16 A alone takes about as long as the device step; a third A buffer gives the
    # copy slack against jitter: equal time on a steady box, profiles/r02/e2e_ab.txt).  With the
    # steady state at max(io_only_ms, device step), the rest of e2e's step is the pipeline's fill
    # (the first H2D) and drain (the last D2H) spread over the steps.
    def run_e2e(es, eflags):
        """es = bytes per host/device element: 4 (uint32 residues, the headline) or 2 (ADJ_IN_U16 |
        ADJ_OUT_U16, phi = T with p < 2^16: half the PCIe bytes each way)."""
        e2e_steps = max(4, args.steps)   # the headline's K: the pipeline's fill and drain amortise alike
        dt = torch.int32 if es == 4 else torch.int16
        hA = torch.empty((m, k * w), dtype=dt, pin_memory=True)
        hA.copy_(A if A.element_size() == es else u32(A))   # residues < 2^16 survive int16 bits
        hC = [torch.empty((m, m * w), dtype=dt, pin_memory=True) for _ in range(2)]
        nA = 3
        dA = [torch.empty((m, k * w), dtype=dt, device=dev) for _ in range(nA)]
        dC = [torch.empty((m, m * w), dtype=dt, device=dev) for _ in range(2)]
        s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        nb = 16                                     # Low(C) read back as nb trapezoidal row blocks
        blocks = [(m * b // nb, m * (b + 1) // nb) for b in range(nb)]
        d2h_bytes = sum((r1 - r0) * r1 * w * es for r0, r1 in blocks)
        ev_in = [torch.cuda.Event() for _ in range(e2e_steps)]
        ev_cmp = [torch.cuda.Event() for _ in range(e2e_steps)]
        ev_out = [torch.cuda.Event() for _ in range(e2e_steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eflags |= flags & ~(adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
        wsz = adj.adjprod_modp_workspace_size(m, k, p, phi, depth, eflags)
        wse = ws if wsz <= ws_bytes else torch.empty(wsz, dtype=torch.uint8, device=dev)
        def d2h(b, stream):
            for r0, r1 in blocks:   # rows [r0, r1) of Low(C) need columns [0, r1) only
                memcpy2d_d2h(hC[b].data_ptr() + r0 * m * w * es, m * w * es,
                             dC[b].data_ptr() + r0 * m * w * es, m * w * es, r1 * w * es, r1 - r0,
                             stream.cuda_stream)

        # the transfers alone: one step's H2D and D2H on their two streams at once, no compute (the
        # copy engines' bound for a step; e2e cannot beat max(this, the device step))
        io = []
        for _ in range(3):
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            c0.record(s_in)
            s_out.wait_event(c0)
            with torch.cuda.stream(s_in):
                dA[0].copy_(hA, non_blocking=True)
            d2h(0, s_out)
            s_in.wait_stream(s_out)
            c1.record(s_in)
            torch.cuda.synchronize()
            io.append(c0.elapsed_time(c1))
        io_ms = statistics.median(io)
        torch.cuda.synchronize()
        t0.record(s_in)
        for i in range(e2e_steps):
            b, a = i % 2, i % nA
            with torch.cuda.stream(s_in):
                if i >= nA:
                    s_in.wait_event(ev_cmp[i - nA])
                dA[a].copy_(hA, non_blocking=True)
                ev_in[i].record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in[i])
                if i >= 2:
                    s_cmp.wait_event(ev_out[i - 2])
                adj.adjprod_modp_ex(m, k, p, phi, dA[a], k, dC[b], m, depth=depth, flags=eflags,
                                    workspace=wse, workspace_bytes=max(wsz, ws_bytes), stream=s_cmp)
                ev_cmp[i].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_cmp[i])
                d2h(b, s_out)
                ev_out[i].record(s_out)
        s_in.wait_stream(s_out)
        t1.record(s_in)
        torch.cuda.synchronize()
        e2e_ms = t0.elapsed_time(t1) / e2e_steps
        last = hC[(e2e_steps - 1) % 2][m - 1, : m * w].numpy()
        last = last.view(np.uint16).astype(np.int64) if es == 2 else last.astype(np.int64)
        ok = bool(np.array_equal(last, u32(C[m - 1, : m * w]).cpu().numpy().astype(np.int64)))
        return {"value": m * m * k / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": hA.numel() * es, "d2h_bytes_per_step": d2h_bytes,
                "h2d_gbs_per_step_time": hA.numel() * es / (e2e_ms * 1e6),   # PCIe-bound: the copy rate
                "d2h_gbs_per_step_time": d2h_bytes / (e2e_ms * 1e6),
                "steps": e2e_steps,
                "pipelined": "3 streams (H2D | C-ABI call | D2H of Low(C) row blocks), 3 A and 2 C buffers",
                "io_only_ms": io_ms,
                "io_only": "one step's H2D and D2H at once on the same streams, no compute (median of 3)",
                "bound_ms": max(io_ms, ms), "frac_of_bound": max(io_ms, ms) / e2e_ms,
                "last_row_matches_device_result": ok}

    # The headline e2e moves residues in the narrowest format the public API accepts for this
    # field: uint16 both ways when phi = T and p < 2^16 (the transfer is PCIe-bound, so this
    # halves it); the uint32 leg is reported beside it as e2e_u32.
    e2e = e2e_u32 = None
    if world == 1:
        # the uint32 leg (context) only where its pinned host buffers stay small (<= 2^27 elements)
        if not io16 or m * k * w <= (1 << 27):
            e2e_u32 = run_e2e(4, 0)
            e2e_u32["io"] = "uint32 residues both ways"
            e2e = e2e_u32
        if io16:
            e2e = run_e2e(2, adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
            e2e["io"] = "uint16 residues both ways (ADJ_IN_U16 | ADJ_OUT_U16)"
    else:
        # N > 1, "A on rank 0": per step rank 0 copies A from pinned host memory,
        # broadcasts it over NCCL, every rank runs adjprod_modp_dist, rank 0 reads Low(C) back;
        # device time per rank, max over ranks
        try:
            e2e_steps = max(3, min(args.steps, 8))
            hA = torch.empty((m, k * w), dtype=A.dtype, pin_memory=True) if rank == 0 else None
            if rank == 0:
                hA.copy_(A)
            hC = torch.empty((m, m * w), dtype=torch.int32, pin_memory=True) if rank == 0 else None
            dA = torch.empty_like(A)
            nb = 16
            blocks = [(m * b // nb, m * (b + 1) // nb) for b in range(nb)]
            d2h_bytes = sum((r1 - r0) * r1 * w * 4 for r0, r1 in blocks)
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            torch.cuda.synchronize()
            t0.record(stream)
            for _ in range(e2e_steps):
                if rank == 0:
                    dA.copy_(hA, non_blocking=True)
                dist.broadcast(dA, src=0)
                adj.adjprod_modp_dist(m, k, p, phi, dA, k, C, m, 0, comm, depth=depth, flags=dist_flags,
                                      stream=stream)
                if rank == 0:
                    for r0, r1 in blocks:
                        memcpy2d_d2h(hC.data_ptr() + r0 * m * w * 4, m * w * 4, C.data_ptr() + r0 * m * w * 4,
                                     m * w * 4, r1 * w * 4, r1 - r0, stream.cuda_stream)
            t1.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([t0.elapsed_time(t1) / e2e_steps], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
            e2e = {"value": m * m * k / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                   "h2d_bytes_per_step": m * k * w * A.element_size(), "d2h_bytes_per_step": d2h_bytes,
                   "steps": e2e_steps,
                   "io": f"A as {'uint16' if A.element_size() == 2 else 'uint32'} from pinned host memory on rank 0, "
                         "NCCL broadcast, uint32 Low(C) read back on rank 0 (SURVEY.md §8(e) 'A on rank 0')"}
        except Exception as ex:  # noqa: BLE001 -- the device-resident line above stands without it
            e2e = {"error": f"{type(ex).__name__}: {ex}"}

    # ---------------- comparators on the same box (context, not the metric): our own depth-0 path
    # (classical int8 SYRK, no Alg. 1 -- the on-box analogue of the paper's classical route,
    # SURVEY.md §8(d)) and cuBLASLt int8 (torch._int_mm) as a library int8 throughput point
    comparators = None
    if world > 1 and dist_mode in ("tiles", "tiles-p2p") and not args.no_compare:
        # the compute-only time of the output-tile sharding -- every rank computes its
        # own regions of Low(C) (adjprod_modp_shard) and leaves them in place, no gather to the root;
        # max over ranks.  Context beside the headline, which includes the gather.
        try:
            fl = dist_flags & ~(adj.ADJ_DIST_TILES | adj.ADJ_DIST_P2P)
            for _ in range(2):
                adj.adjprod_modp_shard(m, k, p, phi, A, k, C, m, rank, world, depth=depth, flags=fl, stream=stream)
            ts = []
            for _ in range(max(3, min(args.steps, 10))):
                flush.zero_()
                dist.barrier()
                a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                adj.adjprod_modp_shard(m, k, p, phi, A, k, C, m, rank, world, depth=depth, flags=fl, stream=stream)
                b0.record(stream)
                torch.cuda.synchronize()
                ts.append(a0.elapsed_time(b0))
            t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            msc = float(t.item())
            comparators = {"compute_only_sharded_output": {
                "ms_per_step": msc, "value": m * m * k / (msc * 1e-3), "unit": UNIT,
                "what": "each rank's owned tile regions of Low(C) computed in place (adjprod_modp_shard), no gather; "
                        "median of flushed steps, max over ranks"}}
            if dist_mode == "tiles-p2p":
                # the same sharding with the NCCL gather (pack, send / recv, unpack) instead of peer stores
                fg = dist_flags & ~adj.ADJ_DIST_P2P
                ts = []
                for i in range(2 + max(3, min(args.steps, 10))):
                    flush.zero_()
                    dist.barrier()
                    a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a0.record(stream)
                    adj.adjprod_modp_dist(m, k, p, phi, A, k, C, m, 0, comm, depth=depth, flags=fg, stream=stream)
                    b0.record(stream)
                    torch.cuda.synchronize()
                    if i >= 2:
                        ts.append(a0.elapsed_time(b0))
                t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                msg = float(t.item())
                comparators["tiles_nccl_gather"] = {
                    "ms_per_step": msg, "value": m * m * k / (msg * 1e-3), "unit": UNIT,
                    "what": "the same output-tile sharding with the result tiles packed, sent to rank 0 with NCCL "
                            "send / recv and unpacked there; median of flushed steps, max over ranks"}
        except Exception as e:  # noqa: BLE001 -- context only, never breaks the headline line
            comparators = {"compute_only_sharded_output": f"unavailable: {type(e).__name__}: {e}"}
    if world == 1 and not args.no_compare:
        comparators = {}

        def other_depth(d, extra=0):
            """the same step at depth d (median of flushed steps) and whether Low(C) is identical"""
            fl = flags | extra
            wsd = adj.adjprod_modp_workspace_size(m, k, p, phi, d, fl)
            wd = torch.empty(max(wsd, 1), dtype=torch.uint8, device=dev)
            Cd = torch.zeros_like(C)
            for _ in range(3):
                adj.adjprod_modp_ex(m, k, p, phi, A, k, Cd, m, depth=d, flags=fl, workspace=wd, workspace_bytes=wsd,
                                    stream=stream)
            ts = []
            for _ in range(max(3, min(args.steps, 10))):
                flush.zero_()
                a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                adj.adjprod_modp_ex(m, k, p, phi, A, k, Cd, m, depth=d, flags=fl, workspace=wd, workspace_bytes=wsd,
                                    stream=stream)
                b0.record(stream)
                torch.cuda.synchronize()
                ts.append(a0.elapsed_time(b0))
            msd = statistics.median(ts)
            lo = torch.tril(torch.ones(m, m, dtype=torch.bool, device=dev))
            same = bool(torch.equal(u32(Cd).view(m, m, w)[lo], u32(C).view(m, m, w)[lo]))
            return {"depth": d, "ms_per_step": msd, "value": m * m * k / (msd * 1e-3), "unit": UNIT,
                    "same_result": same, "workspace_bytes": wsd, "workspace_over_A_bytes": wsd / A_bytes}
        if depth != 0 and not alg1:
            # the classical route (no Alg. 1 level): the on-box analogue of the paper's comparator
            comparators["depth0_classical"] = other_depth(0)
        elif depth == 0 and not alg1 and cfg["phi"] in ("T", "H"):
            # one level of Alg. 1 (inside 2M's G for phi = H) where the automatic depth is 0
            comparators["depth1_alg1"] = other_depth(1)
        if cfg["phi"] == "T" and depth >= 1 and m % 64 == 0:
            # the low-memory temporary schedule (ADJ_LOW_MEM): P1 / P3 / P5 of the root
            # in C's own blocks, the root arena reused by the children, K4 in place
            comparators["low_mem_schedule"] = other_depth(depth, adj.ADJ_LOW_MEM)
        if io16:   # the same step with uint32 residues in HBM
            A4, C4 = u32(A), torch.zeros((m, m * w), dtype=torch.int32, device=dev)
            f4 = flags & ~(adj.ADJ_IN_U16 | adj.ADJ_OUT_U16)
            for _ in range(3):
                adj.adjprod_modp_ex(m, k, p, phi, A4, k, C4, m, depth=depth, flags=f4, workspace=ws,
                                    workspace_bytes=ws_bytes, stream=stream)
            ts = []
            for _ in range(max(3, min(args.steps, 10))):
                flush.zero_()
                a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                adj.adjprod_modp_ex(m, k, p, phi, A4, k, C4, m, depth=depth, flags=f4, workspace=ws,
                                    workspace_bytes=ws_bytes, stream=stream)
                b0.record(stream)
                torch.cuda.synchronize()
                ts.append(a0.elapsed_time(b0))
            ms4 = statistics.median(ts)
            comparators["uint32_residues"] = {"ms_per_step": ms4, "value": m * m * k / (ms4 * 1e-3), "unit": UNIT,
                                              "same_result": bool(torch.equal(torch.tril(C4.view(m, -1)),
                                                                              torch.tril(u32(C).view(m, -1))))}
            del A4, C4
        try:
            n = 8192
            xa = torch.randint(-128, 128, (n, n), dtype=torch.int8, device=dev)
            xb = torch.randint(-128, 128, (n, n), dtype=torch.int8, device=dev)
            for _ in range(3):
                torch._int_mm(xa, xb)
            a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            for _ in range(10):
                torch._int_mm(xa, xb)
            b0.record()
            torch.cuda.synchronize()
            comparators["cublaslt_int8_8192_tops"] = 2.0 * n ** 3 * 10 / (a0.elapsed_time(b0) * 1e-3) / 1e12
            del xa, xb
        except Exception as e:  # noqa: BLE001 -- context only
            comparators["cublaslt_int8_8192_tops"] = f"unavailable: {type(e).__name__}"

    # ---------------- self-check of the timed output on sampled rows.  Not the oracle (bench.py
    # runs oracle/ only in its cpu_baseline / reference legs; parity against the oracle is in
    # tests/test_gpu_fullsize.py at these sizes): the plain definition in int64 numpy, exact
    # since k (p-1)^2 < 2^63, on the last two rows (the longest).
    parity = None
    if rank == 0 and not args.no_check:
        rows = (m - 2, m) if m >= 2 else (0, m)
        Ah = u32(A).cpu().numpy().view(np.uint32).reshape((m, k, w) if w > 1 else (m, k)).astype(np.int64) % p
        got = u32(C).cpu().numpy().view(np.uint32).reshape((m, m, w) if w > 1 else (m, m))
        ok = True
        for i in range(*rows):
            X, Xi = Ah[: i + 1], Ah[i]
            if w == 1:
                ref = [(X @ Xi) % p]
            elif w == 2:   # (x_i + i y_i)(x_j - i y_j) = x_i x_j + y_i y_j + i (y_i x_j - x_i y_j)
                ref = [(X[..., 0] @ Xi[:, 0] + X[..., 1] @ Xi[:, 1]) % p,
                       (X[..., 0] @ Xi[:, 1] - X[..., 1] @ Xi[:, 0]) % p]
            else:          # M_i conj(M_j) by the quaternion table
                a, b, c, d = (Xi[:, q] for q in range(4))
                a2, b2, c2, d2 = (X[..., q] for q in range(4))
                ref = [(a2 @ a + b2 @ b + c2 @ c + d2 @ d) % p,
                       (a2 @ b - b2 @ a + c2 @ d - d2 @ c) % p,
                       (a2 @ c - c2 @ a + d2 @ b - b2 @ d) % p,
                       (a2 @ d - d2 @ a + b2 @ c - c2 @ b) % p]
            for q, r in enumerate(ref):
                g_row = got[i, : i + 1] if w == 1 else got[i, : i + 1, q]
                ok = ok and bool(np.array_equal(g_row.astype(np.int64), r))
        parity = {"rows_checked": list(rows), "bit_exact": ok, "check": "plain definition, int64 numpy"}

    # ---------------- roofline of the dominant kernel (grouped tcgen05 leaf launch)
    peaks, src = load_peaks()
    try:   # which leaf kernel the timed call launches (256 x 256 or the wide 256 x 512 tiles)
        leaf_tile = adj.adjprod_modp_leaf_tile(m, k, p, phi, depth, flags) if world == 1 else 256
    except Exception:  # noqa: BLE001 -- label only
        leaf_tile = None
    leaf_ms, leaf_n = prof_all["leaf"]
    # one grouped leaf stage per step: the tcgen05 leaf launch (+ its tail fixup launch, if any)
    leaf_avg_ms = leaf_ms / args.steps
    ops = leaf_int8_ops(cfg, depth, args.herk) / world   # per GPU: the ranks share the step's leaf work
    achieved = ops / (leaf_avg_ms * 1e-3) / 1e12
    # int8 dense = 2 x bf16 dense (the guide's nominal ratio).  Burst figure for a leaf timed in the
    # burst regime; the sustained (power-capped) figure when the board sat at its power limit during
    # the profiled pass -- a kernel timed inside a long step (B200_PROFILING.md, "Peaks")
    cs = clk_prof.summary() or {}
    capped = ("sw_power_cap" in cs.get("reasons", []) and cs.get("sm_mhz") is not None and cs.get("sm_max_mhz")
              and cs["sm_mhz"] < 0.85 * cs["sm_max_mhz"])   # capped for most of the pass, not a few samples
    bf16 = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) if capped else peaks["bf16_tflops"]
    peak = 2.0 * bf16
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": load_traffic(args.config, depth),
            "kernel": ("leafw_kernel (grouped tcgen05 kind::i8 GEMM/SYRK on 256 x 512 tiles, Horner mod-p "
                       "recombination in TMEM)" if leaf_tile == 512 else
                       "leaf2_kernel (grouped tcgen05 kind::i8 GEMM/SYRK on 256 x 256 tiles + mod-p epilogue)"),
            "peak_source": (f"{src}: 2 x bf16_tflops{'_sustained' if capped else ''} ({bf16}) "
                            f"{'sustained: the board was at its power cap (sw_power_cap) during the timed steps' if capped else 'burst'}"
                            f", int8 = 2x bf16 nominal; of burst (2 x {peaks['bf16_tflops']}): "
                            f"{achieved / (2.0 * peaks['bf16_tflops']):.3f}"),
            "frac_of_spec_dense_int8": achieved / 4500.0,   # B200 datasheet 4.5 POPS dense (context)
            "frac_of_pure_mma_sustained": ((achieved / pm) if capped and (pm := load_pure_mma_sustained()) else None),
            "pure_mma_sustained_source": ("pure tcgen05 kind::i8 issue rate with random operands resident in shared "
                                          "memory, back to back at the power cap on this pool's B200 "
                                          "(profiles/r02/int8_mma_sustained.json, an earlier run)" if capped else None),
            "algorithmic_ops_per_launch": ops, "leaf_ms_per_launch": leaf_avg_ms,
            "leaf_launches_per_step": leaf_n / args.steps,
            "measured": (f"library CUDA events around each leaf launch on the launch stream, over a second "
                         f"pass of the {args.steps} timed steps (same flushes; with these events a step "
                         f"takes {ms_prof:.4f} ms, without them {ms:.4f} ms)"
                         + ("" if world == 1 else
                            f"; N = {world}: 1/N of the step's leaf work over the leaf time averaged over the "
                            f"ranks (each rank runs its share)")),
            "clocks_during": clk_prof.summary()}
    share = {c: round(v[0] / max(1e-9, sum(x[0] for x in prof.values())), 4) for c, v in prof.items()}
    # achieved HBM bandwidth of the HBM-bound kernels (algorithmic bytes / device time per step)
    hb = hbm_bytes(cfg, depth, args.herk, 2 if io16 and world == 1 else 4)
    hbm = None
    if hb is not None:
        hbm = {}
        for cls, nbytes in hb.items():
            t_ms = prof_all[cls][0] / args.steps
            if nbytes is None or t_ms <= 0:
                continue
            gbs = nbytes / world / (t_ms * 1e-3) / 1e9   # N > 1: the single-GPU bytes shared by the ranks
            hbm[cls] = {"bound": "hbm", "algorithmic_bytes": nbytes, "ms": t_ms, "achieved": gbs,
                        "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        Ah = u32(A).cpu().numpy().view(np.uint32).reshape((m, k, w) if w > 1 else (m, k))
        eff, t, cores, desc, _ = oracle_sample(cfg, Ah, float(os.environ.get("ADJ_CPU_BUDGET_S", "10")))
        cpu = {"value": eff, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc, "cpu_model": cpu_model()}

    if rank == 0:
        mh = herk_alg1_macs(m, k) if alg1 else ring_macs(m, k, depth) + {1: 0, 2: 1, 4: 5}[w] * m * m * k
        line = {
            "metric": metric_label(args.config), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "step_ms": step_stats, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic",
            "config": config_dict(args.config, cfg),
            "method": {"depth": depth, "route": ("Alg. 1 over GF(p^2) (ADJ_HERK_ALG1)" if alg1 else
                                                 {"T": "Alg. alg:MIAHMM", "H": "Alg. alg:2M (G through Alg. alg:MIAHMM)",
                                                  "Q": "Alg. alg:2M3M (6M)"}[cfg["phi"]]),
                       "residues": ("uint16 A and Low(C) in HBM (ADJ_IN_U16 | ADJ_OUT_U16)" if io16 and world == 1
                                    else "uint16 A (ADJ_IN_U16), uint32 Low(C) on the root" if io16
                                    else "uint32 A and Low(C) in HBM"),
                       "ring_macs_per_step": mh, "limb_mmas_per_ring_mac": limb_mmas(p),
                       "workspace_bytes": ws_bytes if world == 1 else None,
                       "workspace_over_A_bytes": (ws_bytes / A_bytes) if world == 1 else None},
            "parallelism": ("1 GPU" if world == 1 else
                            (f"output tiles x{world} (NCCL send/recv gather of result tiles)"
                             if dist_mode == "tiles" else
                             f"output tiles x{world} (each rank's final kernel stores its regions into rank 0's C "
                             f"over NVLink)" if dist_mode == "tiles-p2p" else
                             f"split-K x{world} (partials stored into the root over NVLink)"
                             if dist_mode == "p2p" else f"split-K x{world} (NCCL reduce)")),
            "dist_fallback": dist_fallback,
            "fraction_of_int8_peak_effective": value / (world * peak * 1e12 / 2),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "sustained": sustained,
            "e2e_u32": e2e_u32 if (e2e_u32 is not None and e2e is not e2e_u32) else None,
            "gpu_launches": launches,
            "kernel_time_share": share,
            "hbm_kernels": hbm,
            "comparators": comparators,
            "clocks": clk.summary(),
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        adj.adj_comm_destroy(comm)


def relaunch_torchrun(n: int) -> int:
    """`python bench.py --gpus N` outside torchrun: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 with the same arguments; rank 0 prints the JSON line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--depth", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--sustain-s", type=float, default=0.5,
                    help="seconds of back-to-back steps for the sustained (power-capped) context line; 0 = skip")
    ap.add_argument("--io", default="auto", choices=["auto", "u16", "u32"],
                    help="storage of the residues of A and Low(C): auto = uint16 when phi = T, p < 2^16, N = 1")
    ap.add_argument("--no-check", action="store_true", help="skip the sampled parity check")
    ap.add_argument("--no-compare", action="store_true", help="skip the depth-0 / cuBLASLt comparators")
    ap.add_argument("--dist", default="auto", choices=["auto", "splitk", "tiles", "tiles-p2p", "p2p"],
                    help="N > 1: split-K (NCCL reduce), output-tile sharding (NCCL gather of result tiles), "
                         "output-tile sharding with the gather fused into the final kernel (peer stores into the "
                         "root's C over NVLink; auto for square phi = T) or split-K with the exchange fused into "
                         "the final kernel (peer stores into the root's window)")
    ap.add_argument("--herk", default="2m", choices=["2m", "alg1"],
                    help="phi = H: 2M reduction (default) or one level of Alg. 1 over GF(p^2)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        import torch
        if torch.cuda.device_count() < args.gpus:   # one process per GPU: fail before starting ranks
            sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, "
                     f"{torch.cuda.device_count()} visible")
        sys.exit(relaunch_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_gpu(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
