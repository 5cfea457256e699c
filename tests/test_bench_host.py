"""Host-side pieces of bench.py (no GPU): the clock sampler's reduction to the timed region."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class _Done:
    def terminate(self):
        pass

    def wait(self, timeout=None):
        return 0

    def kill(self):
        pass


class _Joined:
    def join(self, timeout=None):
        pass


def _sampler(bench, lines, window):
    s = bench.ClockSampler("0")
    s.proc, s.t = _Done(), _Joined()
    s.lines = lines
    if window is not None:
        s.mark(*window)
    return s.stop()


def _ln(mhz, power_cap=False, thermal=False):
    act = lambda b: "Active" if b else "Not Active"
    return f"{mhz}, 1965, 900.0, Not Active, {act(thermal)}, Not Active, {act(power_cap)}"


def test_only_samples_inside_the_timed_region_count(bench):
    lines = [(0.00, _ln(120)), (0.10, _ln(1965)), (1.00, _ln(1500, power_cap=True)),
             (1.05, _ln(1600, power_cap=True)), (1.10, _ln(1700)), (2.00, _ln(300, thermal=True))]
    c = _sampler(bench, lines, (0.99, 1.12))
    assert c["samples"] == 3
    assert c["sm_mhz"] == 1600
    assert c["reasons"] == ["sw_power_cap"]  # the idle / post-region samples do not leak in


def test_no_sample_inside_falls_back_to_the_nearest_under_load(bench):
    lines = [(0.50, _ln(1800)), (0.90, _ln(1700, power_cap=True)), (3.0, _ln(200))]
    c = _sampler(bench, lines, (1.0, 1.1))
    assert c["samples"] == 2 and c["sm_mhz"] == 1750


def test_no_samples_at_all_is_none(bench):
    assert _sampler(bench, [], (1.0, 1.1)) is None
