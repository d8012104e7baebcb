"""Measured decode profile -> the reference's ProfileTable;
the plateau rule itself is the reference's `estimate_plateau`, unmodified."""
import pytest
from spotrl.balancer import estimate_plateau

from paper_2510_19225_b200.profile import measured_profile_table


def test_measured_table_from_bursts():
    pts = [(1, 10, 0.1, 100.0), (4, 10, 0.1, 300.0), (4, 30, 0.3, 300.0), (2, 0, 0.0, 50.0)]
    t = measured_profile_table(pts)
    assert [(e.batch_size, round(e.decode_throughput, 6)) for e in t.entries] == [(1, 100.0),
                                                                               (4, 400.0)]
    assert t.context_calibration == pytest.approx((100 * 10 + 300 * 40) / 50)


def test_measured_table_feeds_reference_plateau():
    # a B200-like curve: throughput keeps rising to 256, then flattens
    pts = [(b, 100, 100 * (1e-3 + 2e-6 * min(b, 256) + 8e-6 * max(b - 256, 0)), 300.0)
           for b in (1, 64, 128, 256, 384, 512)]
    t = measured_profile_table(pts)
    assert estimate_plateau(t, t.context_calibration) == 256


def test_calibrate_profile_on_fake_instance():
    """The calibration sweep submits b throwaway requests per batch size,
    runs them and keeps the bursts of exactly b rows."""
    from paper_2510_19225_b200.profile import calibrate_profile

    class Inst:
        shape = type("S", (), {"vocab": 50})()

        def __init__(self):
            self.pending = []
            self.done = []

        def decode_profile(self, reset=False):
            out = [(len(self.done), 32, 1e-3 * (1 + 0.01 * len(self.done)), 270.0),
                   (1, 1, 1.0, 270.0)] if self.done else []
            if reset:
                self.done = []
            return out

        def generate(self, rid, prompt, target_len):
            assert len(prompt) == 256 and target_len == 33 and rid.startswith("__calib")
            self.pending.append(rid)

        def run_to_completion(self, n):
            self.done, self.pending = self.pending, []

    t = calibrate_profile(Inst(), [4, 1, 2, 4])
    assert [e.batch_size for e in t.entries] == [1, 2, 4]
    assert t.entries[2].decode_throughput == pytest.approx(4 * 32 / (1e-3 * 1.04))
