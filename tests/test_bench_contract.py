"""Host-side checks of bench.py's launch contract (CPU, no GPU): `--gpus N` never reports a
world size other than N, and the reference arm prints the contract's JSON line."""
import importlib.util
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


class Args:
    def __init__(self, gpus, impl="ours"):
        self.gpus, self.impl = gpus, impl


def test_gpus_must_match_world_size(monkeypatch):
    b = load_bench()
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert b.launch_ranks(Args(8)) == 2          # --gpus 8 under a 4-rank launch: refused
    a = Args(None)
    assert b.launch_ranks(a) is None and a.gpus == 4  # the launcher's world size is taken
    a = Args(4)
    assert b.launch_ranks(a) is None and a.gpus == 4


def test_single_process_defaults(monkeypatch):
    b = load_bench()
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    a = Args(None)
    assert b.launch_ranks(a) is None and a.gpus == 1
    a = Args(8, impl="reference")                # the reference arm runs on rank 0 only
    assert b.launch_ranks(a) is None and a.gpus == 8


def test_reference_arm_line():
    """--impl reference: the oracle on this host's cores, one bounded sample per step."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "samples/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["higher_is_better"] is True


def test_touched_bytes_granules():
    """The roofline's algorithmic bytes: 32-B sectors holding a mapped label,
    and the same over 128-B lines (line_frac); checked against a direct count on a tiny context
    and the ordering sector <= line <= whole row (+ the partial lines of an unaligned row)."""
    import numpy as np
    import bench
    import synth
    spec = synth.ContextSpec(64, [[[0, 9, 40], [63]]], 0.0, 10.0)  # one app: f32 columns 0, 9, 40, 63
    # rows of 64 f32 = 256 B (sector / line aligned): sectors {0, 1, 5, 7}, lines {0, 1}
    assert bench.touched_sector_bytes(spec, 64, 4) == 4 * 32
    assert bench.touched_sector_bytes(spec, 64, 4, granule=128) == 2 * 128
    for cfg in (2, 3, 4):
        sp = synth.config_context(cfg)
        ld = synth.default_ld(sp.C, "f32")
        s = bench.touched_sector_bytes(sp, ld, 4, rows=1 << 20)
        ln = bench.touched_sector_bytes(sp, ld, 4, rows=1 << 20, granule=128)
        assert 0 < s <= ln <= ld * 4 + 128, (cfg, s, ln)
    assert np.isclose(bench.touched_sector_bytes(synth.config_context(2), 1000, 4), 3168.0)
