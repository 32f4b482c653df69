"""bench.py contract checks that run without a GPU: the reference arm's JSON
line (the CPU oracle on a bounded sample; the driver launches this arm
exactly like ours) and the clock sampler's summary when no GPU is visible."""
import json
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "small",
                        "--steps", "1", "--warmup", "3", "--cpu-budget", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "Gvoxels/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["cpu_baseline"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "Gvoxels/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["field"] == [256, 256, 256]


def test_clock_sampler_without_gpu():
    sys.path.insert(0, str(ROOT))
    import bench

    with bench.ClockSampler(0) as clk:
        pass
    s = clk.summary()
    assert set(s) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert isinstance(s["reasons"], list)
