"""The GPU-path harness and CLI (reference harness.py / cli.py; SURVEY.md §8f
item 3): synthetic streams pinned to the reference's own output, CLI
plumbing on CPU, replay / bench / breakdown on the GPU."""

import json
import os

import numpy as np
import pytest
import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden_synth():
    return np.load(os.path.join(HERE, "golden", "synth.npz"))


def test_synth_streams_match_reference():
    from paper_2504_03661_b200.harness import SynthSpec, synth_kv
    g = _golden_synth()
    specs = [dict(n_tokens=64, d=128, seed=0),
             dict(n_tokens=50, d=128, seed=3, outlier_channels=[7, 63]),
             dict(n_tokens=40, d=64, seed=9, sigma=0.5, outlier_channels=[1],
                  outlier_rate=0.01, outlier_magnitude=30.0)]
    for si, sp in enumerate(specs):
        K, V = synth_kv(SynthSpec(**sp))
        np.testing.assert_array_equal(K, g[f"s{si}_K"])
        np.testing.assert_array_equal(V, g[f"s{si}_V"])


def test_synth_spec_validation():
    from paper_2504_03661_b200.harness import SynthSpec
    with pytest.raises(ValueError):
        SynthSpec(n_tokens=4, d=8, outlier_channels=[8])
    with pytest.raises(ValueError):
        SynthSpec(n_tokens=4, sigma=0.0)
    with pytest.raises(ValueError):
        SynthSpec(n_tokens=4, outlier_rate=1.0)


def test_cli_synth_writes_reference_format(tmp_path):
    from click.testing import CliRunner
    from paper_2504_03661_b200 import cli, fileio
    r = CliRunner().invoke(cli.main, ["synth", "--n-tokens", "16", "--d", "32", "--seed", "2",
                                      "--outlier-channels", "3,5", "--out", str(tmp_path)])
    assert r.exit_code == 0, r.output
    K = fileio.read_tensor(tmp_path / "keys.f32")
    assert K.shape == (16, 32) and K.dtype == np.float32


def test_cli_bad_preset_and_config_key(tmp_path):
    from click.testing import CliRunner
    from paper_2504_03661_b200 import cli
    r = CliRunner().invoke(cli.main, ["bench", "--preset", "nope", "--out", str(tmp_path)])
    assert r.exit_code != 0
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"no_such_option": 1}))
    r = CliRunner().invoke(cli.main, ["synth", "--config", str(cfg), "--out", str(tmp_path)])
    assert r.exit_code != 0


def _stream_and_codebooks(tmp_path, n=96, seed=4):
    from paper_2504_03661_b200 import fileio
    from paper_2504_03661_b200.harness import SynthSpec, sampled_codebooks, synth_kv
    from paper_2504_03661_b200.pq_core import PQConfig
    K, V = synth_kv(SynthSpec(n_tokens=n, d=128, seed=seed, outlier_channels=[7]))
    cbk, cbv = sampled_codebooks(*synth_kv(SynthSpec(n_tokens=512, d=128, seed=1)),
                                 PQConfig(128, 64, 8))
    fileio.write_tensor(tmp_path / "k.f32", K)
    fileio.write_tensor(tmp_path / "v.f32", V)
    fileio.write_codebook(tmp_path / "ck.pqkv", cbk)
    fileio.write_codebook(tmp_path / "cv.pqkv", cbv)
    return K, V, cbk, cbv


@pytest.mark.gpu
@pytest.mark.parametrize("recent,flush", [(0, 1), (16, 16)])
def test_verify_stream_gpu(tmp_path, recent, flush):
    from paper_2504_03661_b200.harness import verify_stream
    K, V, cbk, cbv = _stream_and_codebooks(tmp_path)
    rep = verify_stream(K, V, cbk, cbv, recent_capacity=recent, flush_threshold=flush,
                        n_prefill=40)
    assert rep["steps"] == 56 and rep["max_rel_error"] <= 1e-5, rep


@pytest.mark.gpu
def test_cli_verify_bench_breakdown_gpu(tmp_path):
    from click.testing import CliRunner
    from paper_2504_03661_b200 import cli
    _stream_and_codebooks(tmp_path)
    run = CliRunner().invoke
    r = run(cli.main, ["verify", "--keys", str(tmp_path / "k.f32"), "--values",
                       str(tmp_path / "v.f32"), "--cb-key", str(tmp_path / "ck.pqkv"),
                       "--cb-value", str(tmp_path / "cv.pqkv"), "--out", str(tmp_path)])
    assert r.exit_code == 0 and "PASS" in r.output, r.output
    r = run(cli.main, ["bench", "--contexts", "256,512", "--gen-tokens", "3", "--repetitions",
                       "3", "--warmup", "0", "--seed", "0",
                       "--out", str(tmp_path)])
    assert r.exit_code == 0, r.output
    rows = (tmp_path / "bench.csv").read_text().splitlines()
    assert rows[0] == ",".join(cli.BENCH_CSV_COLUMNS) and len(rows) == 3
    r = run(cli.main, ["breakdown", "--contexts", "512", "--gen-tokens", "3", "--worker", "sync",
                       "--out", str(tmp_path)])
    assert r.exit_code == 0, r.output
    assert (tmp_path / "breakdown.csv").read_text().splitlines()[0] == \
        ",".join(cli.BREAKDOWN_CSV_COLUMNS)


@pytest.mark.gpu
def test_cli_train_matches_reference_training(tmp_path):
    """`train` (cli.py:108-155) on the golden training samples writes the
    reference's codebook bit for bit (tests/golden/kmeans.npz, made by running
    the reference's train_codebooks)."""
    import os
    from click.testing import CliRunner
    from paper_2504_03661_b200 import cli, fileio
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "kmeans.npz"))
    fileio.write_tensor(tmp_path / "k.f32", g["train_X"])
    fileio.write_tensor(tmp_path / "v.f32", g["train_X"])
    r = CliRunner().invoke(cli.main, ["train", "--keys", str(tmp_path / "k.f32"), "--values",
                                      str(tmp_path / "v.f32"), "--m", "8", "--nbits", "4",
                                      "--kmeans-iters", "12", "--seed", "7",
                                      "--out", str(tmp_path)])
    assert r.exit_code == 0, r.output
    assert "bits_per_value" in r.output and "per-subspace distortion" in r.output
    cb = fileio.read_codebook(tmp_path / "cb_key.pqkv")
    np.testing.assert_array_equal(cb.centroids, g["train_C"])
    assert fileio.read_codebook(tmp_path / "cb_value.pqkv").kind == "value"


@pytest.mark.gpu
def test_cli_sensitivity_and_stats(tmp_path):
    """`sensitivity` / `stats` (cli.py:307-366): the reference's options, JSON
    files and echo lines, backed by analysis.py (pinned by analysis.npz)."""
    import json
    import os
    from click.testing import CliRunner
    from paper_2504_03661_b200 import analysis, cli, fileio
    from paper_2504_03661_b200.pq_core import PQConfig
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "analysis.npz"))
    fileio.write_tensor(tmp_path / "k.f32", g["X"])
    run = CliRunner().invoke
    r = run(cli.main, ["stats", "--keys", str(tmp_path / "k.f32"), "--out", str(tmp_path)])
    assert r.exit_code == 0 and "global absmax" in r.output, r.output
    st = json.loads((tmp_path / "stats.json").read_text())
    np.testing.assert_allclose(st["absmax"], g["cs_absmax"], rtol=1e-12)
    r = run(cli.main, ["sensitivity", "--keys", str(tmp_path / "k.f32"), "--m", "16",
                       "--nbits", "4", "--seed", "2", "--out", str(tmp_path)])
    assert r.exit_code == 0 and "pq sensitivity" in r.output, r.output
    rep = json.loads((tmp_path / "sensitivity.json").read_text())
    assert set(rep) == {"fraction", "bits_per_value", "pq", "int"}
    want = analysis.sensitivity_study(g["X"], PQConfig(32, 16, 4, seed=2), fraction=0.01)
    assert rep["pq"]["sensitivity"] == pytest.approx(want.sensitivity, rel=1e-12)
