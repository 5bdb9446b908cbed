"""bench.py's measurement helpers on the CPU: the energy window average against the
reference's own haloflow.energy.window_average (energy.py:83-111), the refusal to
run with kernel-skipping debug switches, identical config keys in both arms."""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def _reference_energy():
    ref = Path("/root/reference/pkg/src")
    if not ref.exists():
        pytest.skip("reference sources not present (GPU box)")
    sys.path.insert(0, str(ref))
    from haloflow import energy

    return energy


@pytest.mark.parametrize("t0,t1", [(0.0, 1.0), (0.05, 0.35), (-1.0, 2.0), (0.3, 0.31)])
def test_window_average_matches_reference(t0, t1):
    energy = _reference_energy()
    samples = [(0.0, 100.0), (0.1, 250.0), (0.25, 400.0), (0.3, 150.0), (0.9, 500.0)]
    ref = energy.window_average([energy.PowerSample(t, w) for t, w in samples], t0, t1)
    assert bench.window_average(samples, t0, t1) == pytest.approx(ref, rel=1e-15, abs=1e-12)


def test_refuses_debug_switches(monkeypatch):
    monkeypatch.setenv("SHT_FFT_DEBUG", "1")
    with pytest.raises(SystemExit):
        bench.refuse_debug()
    monkeypatch.setenv("SHT_FFT_DEBUG", "0")
    bench.refuse_debug()


def test_both_arms_report_the_same_config():
    class A:
        truncation, nfld = 639, 548

    cfg = bench.config_of(A())
    assert cfg == {"workload": "TCo639 inverse+direct pair, 548 fields", "truncation": 639, "nfld": 548,
                   "grid": "octahedral"}
