"""bench.py's roofline arithmetic (host only) reproduces SURVEY.md §8(d)'s worked numbers:
M2 at d=1 (T2 = 10.0 ms, T3 = 20.5 ms) and M3 Llama-3.1-70B at d=8, B=256, S_ctx=1700
(T2 = T3 = 133.4 ms), with the survey's peaks (1634.2 TFLOP/s, 6549.1 GB/s, NVLink 900 GB/s)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from sidp_inputs import MODELS  # noqa: E402

PEAKS = {"tflops": 1634.2, "hbm": 6549.1, "nvl": 900.0}


def test_m2_single_gpu_t2_t3():
    r = bench.north_star_roofline(MODELS["qwen3-32b"], 256, 1024, 1, PEAKS, step_ms=1.0)
    assert r["T2_ms"] == pytest.approx(10.0, abs=0.05)
    assert r["T3_ms"] == pytest.approx(20.5, abs=0.05)
    assert r["nvlink_bytes_per_step"] == 0.0


def test_m3_llama_d8_t2_equals_t3():
    m = MODELS["llama-3.1-70b"]
    r = bench.north_star_roofline(m, 256, 1700, 8, PEAKS, step_ms=1.0)
    assert r["T2_ms"] == pytest.approx(133.4, abs=0.1)
    assert r["T3_ms"] == pytest.approx(133.4, abs=0.1)
    # 70 remote layers of 1.7113 GB per step (119.8 GB)
    assert r["nvlink_bytes_per_step"] == pytest.approx(119.8e9, rel=2e-3)


def test_remote_bytes_override_and_kernel_work():
    m = MODELS["qwen3-32b"]
    r = bench.north_star_roofline(m, 256, 1024, 8, PEAKS, 1.0, remote_bytes=44e9)
    assert r["nvlink_bytes_per_step"] == 44e9
    # attention: 4096 B of K/V per context token per layer (+ q and o), 2 x 2 x n_q hd flops
    fl, by = bench.kernel_work(2, m, 256, 1024, 0)
    assert by == pytest.approx(2.0 * 2 * m.kv_dim * 256 * 1025 + 2.0 * 2 * 256 * m.q_dim)
    assert fl == pytest.approx(4.0 * m.n_q_heads * m.head_dim * 256 * 1025)


def test_fused_mlp_kernel_work():
    """The fused gate/up -> down launch (mlp2_kernel) is charged both GEMMs' work: 2 B (2I) h +
    2 B h I flops (Qwen3-32B at B = 256: 201.3 GFLOP) and the three weight matrices once."""
    m = MODELS["qwen3-32b"]
    B, h, I = 256, m.hidden, m.intermediate
    fl, by = bench.kernel_work(1, m, B, 0, 0, fused_mlp=True)
    fl_gu, _ = bench.kernel_work(1, m, B, 0, 0)
    fl_d, _ = bench.kernel_work(4, m, B, 0, 0)
    assert fl == pytest.approx(fl_gu + fl_d)
    assert fl == pytest.approx(201.3e9, rel=1e-3)
    # + the act tile written and read once (B I bf16 x 2, 3.3% at B = 256), x in, fp32 slice out
    assert by >= 2.0 * 3 * I * h and by < 2.0 * 3 * I * h * 1.05
