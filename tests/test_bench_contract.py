"""bench.py's driver contract on the host: the reference arm (the CPU oracle timed as it stands,
DESIGN.md §7) prints one JSON line with the contract's keys, and the bench's own bookkeeping
(ring MAC counts, algorithmic bytes) follows the closed forms of Alg. alg:MIAHMM."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_json_line():
    env = dict(os.environ, ADJ_REF_STEP_S="0.05")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, env=env, timeout=300,
                         cwd=ROOT, check=True).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["metric"] == bench.metric_label("c1") and d["unit"] == bench.UNIT
    assert d["value"] > 0 and d["higher_is_better"] is True and d["steps"] == 2
    # the same config dict the GPU arm prints (what is computed, not how)
    assert d["config"] == bench.config_dict("c1", bench.CONFIGS["c1"])
    assert d["config"]["workload"] == bench.CONFIGS["c1"]["workload"]
    # ms_per_step is the measured slab time; the extrapolation to the full problem is reported apart
    assert 0 < d["ms_per_step"] <= d["extrapolated_full_problem_ms"] * 1.0001
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_ring_macs_leading_ratios():
    """R_d / R_0 -> (7/8)^... : one level of Alg. 1 does 3 half-size SYRKs and 2 half-size
    general products, 7/8 of the classical lower-triangle MACs as m, k grow;
    two levels 53/64."""
    m = k = 1 << 20
    r0 = bench.ring_macs(m, k, 0)
    assert abs(bench.ring_macs(m, k, 1) / r0 - 7 / 8) < 1e-5
    assert abs(bench.ring_macs(m, k, 2) / r0 - 53 / 64) < 1e-5
    # exact small case: m = k = 2, one level = 3 (1x1 SYRK, k = 1) + 2 (1x1x1) = 5 MACs
    assert bench.ring_macs(2, 2, 1) == 5


@pytest.mark.parametrize("res_bytes", [2, 4])
def test_hbm_bytes_c2(res_bytes):
    """K1 at c2 depth 1: A read once, 7 operands x 3 limb planes of (m/2) x (k/2) int8 written;
    K4: P1, P2, P5 lower + P3, P4 full uint16 read once, Low(C) written once."""
    cfg = bench.CONFIGS["c2"]
    m, k = cfg["m"], cfg["k"]
    hb = bench.hbm_bytes(cfg, 1, res_bytes=res_bytes)
    mh, kh = m // 2, k // 2
    assert hb["preadd"] == res_bytes * m * k + 7 * 3 * mh * kh
    assert hb["combine"] == (3 * mh * (mh + 1) // 2 + 2 * mh * mh) * 2 + m * (m + 1) // 2 * res_bytes


@pytest.mark.gpu
def test_gpu_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "3",
                          "--warmup", "3", "--no-cpu", "--no-compare"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT, check=True).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["metric"] == bench.metric_label("c1") and d["n_gpus"] == 1
    assert d["config"] == bench.config_dict("c1", bench.CONFIGS["c1"]) and d["steps"] == 3 and d["warmup"] >= 3
    assert d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["last_row_matches_device_result"]
    assert d["parity"]["bit_exact"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_hbm_bytes_c3_depth2():
    """K1 / K4 algorithmic bytes at c3 depth 2 (the N = 1 headline) written out level by level:
    level 1 reads A once and writes 4 operands (S1, S2, S4, X22) x 2 planes plus S3 (uint16);
    level 2 has 3 nodes (A11, A12 views of A and S3) each writing 7 operands x 2 planes; K4 reads
    3 lower + 2 full product buffers per node and writes Low of its output.  With uint16 residues
    the library fuses K1 of levels 1 and 2 (one read of A, S3 kept in registers): no level-2 reads
    and no S3 round trip."""
    cfg = bench.CONFIGS["c3"]
    n = cfg["m"]
    assert cfg["k"] == n
    h1, h2 = n // 2, n // 4
    for rb in (2, 4):
        hb = bench.hbm_bytes(cfg, 2, res_bytes=rb)
        if rb == 4:
            pre = (rb * n * n + 4 * 2 * h1 * h1 + 2 * h1 * h1               # level 1
                   + 2 * h1 * h1 * rb + h1 * h1 * 2 + 3 * 7 * 2 * h2 * h2)    # level 2: reads, writes
        else:
            pre = rb * n * n + 4 * 2 * h1 * h1 + 3 * 7 * 2 * h2 * h2          # fused levels 1 + 2
        comb = (3 * ((3 * h2 * (h2 + 1) // 2 + 2 * h2 * h2) * 2 + h1 * (h1 + 1) // 2 * 2)
                + (3 * h1 * (h1 + 1) // 2 + 2 * h1 * h1) * 2 + n * (n + 1) // 2 * rb)
        assert hb == {"preadd": pre, "combine": comb}


def test_metric_label_names_the_config():
    assert bench.DEFAULT_CONFIG == "c3"
    assert "c3: BASELINE configs[2]" in bench.metric_label("c3")
    assert "c4: BASELINE configs[3]" in bench.metric_label("c4")


def test_hbm_bytes_compact_halves_the_residue_terms():
    """Only the caller-residue terms (reading A, writing Low(C)) shrink with uint16 storage; the
    limb planes and the narrow product buffers do not."""
    for name, depth in (("c2", 0), ("c2", 1), ("c5", 0), ("q5", 0)):
        cfg = bench.CONFIGS[name]
        m, k = cfg["m"], cfg["k"]
        w = {"T": 1, "H": 2, "Q": 4}[cfg["phi"]]
        b4, b2 = bench.hbm_bytes(cfg, depth, res_bytes=4), bench.hbm_bytes(cfg, depth, res_bytes=2)
        assert b4["preadd"] - b2["preadd"] == 2 * w * m * k
        if b4["combine"] is not None:
            assert b4["combine"] - b2["combine"] == 2 * w * m * (m + 1) // 2


def test_bench_help():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                         cwd=ROOT, timeout=120, check=True).stdout
    for flag in ("--gpus", "--steps", "--warmup", "--config", "--impl", "--io", "--dist", "--sustain-s"):
        assert flag in out
