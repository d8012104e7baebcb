"""bench.py pieces that run without a GPU: the clocks summary (median SM
clock under load, throttle reasons) and the CLI defaults of the contract."""
import sys

import bench


def test_clock_summary_under_load():
    cs = bench.ClockSampler(0)
    cs.rows = [["1965", "1965", "Not Active", "Not Active", "Not Active", "Not Active", "3"],
               ["1815", "1965", "Not Active", "Not Active", "Not Active", "Active", "99"],
               ["1830", "1965", "Not Active", "Not Active", "Not Active", "Active", "98"],
               ["1800", "1965", "Not Active", "Not Active", "Not Active", "Not Active", "97"],
               ["garbage"]]
    s = cs.summary()
    assert s["sm_mhz"] == 1815 and s["sm_max_mhz"] == 1965
    assert s["reasons"] == ["sw_power_cap"] and s["samples"] == 3


def test_clock_summary_unsampled():
    assert bench.ClockSampler(0).summary()["reasons"] == ["unsampled"]


def test_cli_defaults(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert (a.gpus, a.steps, a.impl) == (1, 2, "b200") and a.warmup >= 3
    assert a.prompts == 512 and a.new_tokens == 1024 and not a.strong
