"""bench.py contract checks that run without a GPU: the reference arm (CPU
oracle on a bounded sample) prints one well-formed JSON line."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_contract_line():
    out = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config",
         "bootstrap", "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=600, cwd=REPO,
    )
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "CKKS bootstrap ms (N=2^16)" and line["unit"] == "ms"
    assert line["higher_is_better"] is False
    assert line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run(
        [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1",
         "--warmup", "0"],
        capture_output=True, text=True, timeout=120, cwd=REPO, env=env,
    )
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_clock_summary_flags_throttle_reasons():
    """The clocks object of the bench line: median SM clock under load, max
    clock, and every throttle reason seen in any sample (rows as the NVML and
    nvidia-smi samplers record them)."""
    sys.path.insert(0, REPO)
    import bench

    c = bench.ClockSampler(0)
    c.samples = [["1965", "1965", "", "Not Active", "Not Active", "Not Active", "Not Active"],
                 ["1950", "1965", "", "Not Active", "Not Active", "Not Active", "Active"],
                 ["1965", "1965", "", "Active", "Not Active", "Not Active", "Not Active"]]
    s = c.summary()
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0 and s["samples"] == 3
    assert s["reasons"] == ["hw_slowdown", "sw_power_cap"]
    assert bench.ClockSampler(0).summary()["reasons"] == ["unsampled"]
