"""bench.py host logic on CPU: the reference arm's JSON line (the driver
parses it), the CPU-arm sample and its reference/port equivalence, and the
roofline helpers."""

import json
import sys
import types

import numpy as np
import pytest

import bench
import paper_2406_18820_b200 as U


def _args(**kw):
    base = dict(gpus=1, steps=1, warmup=0, impl="reference", config="cfg1", layers=2,
                cpu_threads=2)
    base.update(kw)
    return types.SimpleNamespace(**base)


def test_reference_arm_json_line(capsys):
    bench.run_reference(_args())
    line = capsys.readouterr().out.strip().splitlines()[-1]
    d = json.loads(line)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["config"]["workload"]


def test_reference_arm_other_ranks_do_nothing(capsys, monkeypatch):
    monkeypatch.setenv("RANK", "1")
    bench.run_reference(_args())
    assert capsys.readouterr().out == ""


def test_cpu_arm_reference_and_port_agree():
    spec, src, tgt, _ = U.bench_config("cfg1", 2)
    names = bench.sample_params(spec, 1e8)
    assert names and all(n.startswith("layers.") for n in names)
    frags = bench.oracle_frags(spec, src, names, 2)
    outs = {}
    for prefer in (True, False):
        arm = bench.CpuArm(spec, src, tgt, frags, prefer)
        got = {}
        assert arm.run(2, got) > 0
        outs[arm.kind] = got
    if "reference" not in outs:
        pytest.skip("reference package not staged")
    a, b = outs["reference"], outs["port"]
    assert a.keys() == b.keys() and a
    for k in a:
        assert np.array_equal(np.asarray(a[k]).view(np.uint8), np.asarray(b[k]).view(np.uint8)), k


def test_link_roofline_and_peak_fallback(tmp_path, monkeypatch):
    link = {"h2d_GBps": 50.0, "d2h_GBps": 50.0, "bidir_GBps": 100.0}
    r = bench.link_roofline(link, 10 ** 9, 10 ** 9, 40.0)
    assert r["achieved_GBps"] == pytest.approx(50.0) and r["frac"] == pytest.approx(0.5)
    assert bench.link_roofline({}, 1, 1, 1.0) == {}
    # the step's own byte mix pushed through the link alone: 1 GB of H2D
    # (with its D2H alongside) takes 20 ms, so a 40 ms step is at 0.5
    mixed = dict(link, mixed={"d2h_per_h2d": 1.0, "s_per_h2d_byte": 0.02 / 10 ** 9})
    m = bench.link_roofline(mixed, 10 ** 9, 10 ** 9, 40.0)["mixed"]
    assert m["bound_ms"] == pytest.approx(20.0) and m["frac"] == pytest.approx(0.5)
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    peak, src = bench.measured_peak()
    assert peak > 0 and src.startswith("fallback")
