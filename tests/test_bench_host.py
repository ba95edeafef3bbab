"""Host-side pieces of bench.py (no GPU): clock-sample parsing and the timed-window selection."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import pytest  # noqa: E402


def _line(sm, smax=1965, power_cap="Not Active", thermal="Not Active"):
    return f"0, {sm}, {smax}, 700.0, 0x0, Not Active, Not Active, {thermal}, {power_cap}\n"


def test_clock_summary_uses_timed_window_and_reasons():
    c = bench.ClockSampler(0)
    c.samples = [(0.0, _line(1200)), (1.0, _line(1965)), (1.1, _line(1950, power_cap="Active")),
                 (5.0, _line(900, thermal="Active"))]
    c.t0, c.t1 = 0.9, 1.2
    s = c.summary()
    assert s["window"] == "timed" and s["samples"] == 2
    assert s["sm_mhz"] == 1957.5 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]


def test_clock_summary_falls_back_to_whole_run():
    c = bench.ClockSampler(0)
    c.samples = [(0.0, _line(1965)), (0.5, "garbage\n")]
    c.t0, c.t1 = 2.0, 2.1
    s = c.summary()
    assert s["window"] == "run" and s["samples"] == 1 and s["sm_mhz"] == 1965.0


def test_flop_and_byte_model_matches_survey_appendix_b():
    from paper_0901_1024_b200.perfmodel import bytes_per_element_stage, flops_per_element_stage

    assert flops_per_element_stage(4) == 76410 and flops_per_element_stage(6) == 381864
    assert bytes_per_element_stage(4, 4) == 3496 and bytes_per_element_stage(9, 4) == 21256


@pytest.mark.parametrize("data,want,key", [
    ({"hbm_gbs": 6535.2, "bf16_tflops": 1500.0}, 6535.2, "hbm_gbs"),
    ({"hbm": {"copy_gbs_burst": 6800.0, "copy_gbs_sustained": 6535.0}}, 6535.0, "hbm.copy_gbs_sustained"),
    ({"dram_tbs": 6.5}, 6500.0, "dram_tbs"),
])
def test_measured_peaks_parsing(tmp_path, monkeypatch, data, want, key):
    """bench._peaks reads the driver-written MEASURED_PEAKS.json whatever its key layout."""
    import json

    import bench

    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    assert bench._peaks()["_fallback"]
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps(data))
    got = bench._peaks()
    assert got["hbm_gbs"] == pytest.approx(want) and got["source"].endswith(key)


@pytest.mark.parametrize("order,word,path,bound", [(4, 4, "tensor", "hbm"), (4, 8, "simt", "fp64"),
                                                   (9, 4, "tensor", "tensor"), (7, 8, "simt", "fp64"),
                                                   (1, 4, "simt", "hbm"), (4, 4, "tensor2", "hbm")])
def test_roofline_model_names_the_binding_term(order, word, path, bound):
    """T_roof = max(B_alg / BW, F_alg / P) with P the pipe the kernel computes on."""
    peaks = {"hbm_gbs": 6548.8, "source": "test"}
    pipes = {"fp32_tflops": 74.4, "fp64_tflops": 37.2,
             "tf32": {"tflops": 1152.0, "source": "test"},
             "fp64": {"dmma_tflops": 37.1, "dfma_tflops": 36.0, "source": "test"}}
    r = bench.roofline(order, word, path, 998250, 1e-3, peaks, pipes, "k", None)
    assert r["bound"] == bound
    assert r["frac"] == pytest.approx(max(r["hbm_term_us"], r["compute_term_us"]) / 1e3)
    assert r["unit"] == ("GB/s" if bound == "hbm" else "TFLOP/s")
    pipes_no_probe = dict(pipes, tf32=None, fp64=None)
    assert bench.roofline(order, word, path, 998250, 1e-3, peaks, pipes_no_probe, "k", None)["frac"] > 0
