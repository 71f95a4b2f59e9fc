"""The `vqkv` CLI (tools/vqkv_cli.cpp, f2) and the GPU trainer (trainer.cu, f4).

* CPU: the host-only subcommands (ratio, stats --config, gen) against the reference's own expected
  output (proj/tests/cli_pipeline.cmake:26-42) and the oracle's generator.
* GPU: the port of cli_pipeline.cmake (ratio -> stats -> gen -> train -> compress -> bench, the same
  regexes), with the trained stacks, the VQCM codes and the loss reports checked against the oracle's
  restatement of trainer.cpp / codebook.cpp; and one trainer batch (D = 128) bit for bit.
"""
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cli():
    from paper_2603_16435_b200 import build

    return build.build_cli()


def run(cli, *args):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True)
    assert r.returncode == 0, f"vqkv {' '.join(map(str, args))} failed ({r.returncode}):\n{r.stdout}\n{r.stderr}"
    return r.stdout


def test_cli_ratio_stats_gen(cli, tmp_path):
    assert "82.8%" in run(cli, "ratio", "--nk", 56, "--sk", 1024, "--nv", 16, "--sv", 512)
    assert re.search(r"percent=82\.4", run(cli, "stats", "--config", "56,1024,10,65536", "--precise"))
    out = run(cli, "gen", "--kind", "rope_rotated_keys", "--dim", 16, "--count", 500, "--components", 4, "--std",
              0.2, "--seed", 7, "--out", tmp_path / "k.vecd")
    assert out.startswith("gen kind=rope_rotated_keys dim=16 count=500 ")
    b = (tmp_path / "k.vecd").read_bytes()
    assert b[:4] == b"VECD" and np.frombuffer(b[4:8], np.uint32)[0] == 1
    x = np.frombuffer(b[20:], np.float32).reshape(500, 16)
    assert np.array_equal(x, O.generate(O.ROPE_ROTATED_KEYS, 16, 500, 4, 7, component_std=0.2))
    r = subprocess.run([cli, "ratio", "--nk", "1"], capture_output=True, text=True)
    assert r.returncode != 0 and "required" in r.stderr


def read_vecd(p):
    b = open(p, "rb").read()
    d, n = np.frombuffer(b[8:12], np.uint32)[0], np.frombuffer(b[12:20], np.uint64)[0]
    return np.frombuffer(b[20:], np.float32).reshape(int(n), int(d))


@pytest.mark.gpu
def test_cli_pipeline_vs_oracle(cli, tmp_path):
    """cli_pipeline.cmake:26-76 on the GPU build, then the artefacts against the oracle."""
    w = tmp_path
    assert "82.8%" in run(cli, "ratio", "--nk", 56, "--sk", 1024, "--nv", 16, "--sv", 512)
    assert re.search(r"percent=82\.4", run(cli, "stats", "--config", "56,1024,10,65536", "--precise"))
    run(cli, "gen", "--kind", "gaussian_mixture", "--dim", 16, "--count", 8000, "--components", 8, "--std", 0.1,
        "--seed", 41, "--out", w / "keys.vecd")
    run(cli, "gen", "--kind", "gaussian_mixture", "--dim", 16, "--count", 8000, "--components", 8, "--std", 0.1,
        "--seed", 42, "--out", w / "values.vecd")
    out = run(cli, "train", "--data", w / "keys.vecd", "--stages", "32,32,32", "--epochs", 40, "--lr", 0.01, "--seed", 1,
              "--kind", "key", "--out", w / "key.rsvq")
    assert "train final_mse=" in out
    run(cli, "train", "--data", w / "values.vecd", "--stages", "32,32,32", "--epochs", 40, "--lr", 0.01, "--seed", 2,
        "--kind", "value", "--out", w / "value.rsvq")
    out_c = run(cli, "compress", "--data", w / "keys.vecd", "--stack", w / "key.rsvq", "--out", w / "keys.vqcm")
    assert "compress rows=8000 " in out_c
    assert (w / "keys.vqcm").exists()
    out_b = run(cli, "bench", "--spec", "kind=gaussian_mixture,components=8,seed=41,std=0.1", "--key-stack",
                w / "key.rsvq", "--value-stack", w / "value.rsvq", "--linit", 4, "--llocal", 128, "--tokens", 1536,
                "--prefill", 1024, "--queries", 32, "--block-rows", 64, "--checkpoint", 256)
    assert "checkpoint tokens=1536 " in out_b
    assert re.search(r"output_mean_cosine=(1\.0|0\.99)", out_b), out_b
    assert "within_budget=1" in out_b

    # trainer parity: the CLI's stack (GPU batches) == the oracle's trainer.cpp restatement, bit for bit
    keys = read_vecd(w / "keys.vecd")
    cfg = O.train_config(learning_rate=0.01, epochs=40, seed=1)
    ost, eloss, smse = O.train(keys, [32, 32, 32], cfg, O.KEY)
    gst = O.Stack.load(str(w / "key.rsvq"))
    for s in range(3):
        assert np.array_equal(gst.projection(s), ost.projection(s)), f"stage {s} projection differs"
        assert np.array_equal(gst.entries(s), ost.entries(s))
    got_epochs = [float(m) for m in re.findall(r"epoch index=\d+ loss=(\S+)", out)]
    assert np.allclose(got_epochs, eloss, rtol=1e-6, atol=0)
    final = float(re.search(r"train final_mse=(\S+)", out).group(1))
    assert abs(final - smse[-1]) <= 1e-6 * abs(smse[-1])
    # compress parity: VQCM codes == the oracle's quantize_batch with the same stack
    b = (w / "keys.vqcm").read_bytes()
    assert b[:4] == b"VQCM"
    ref_pay, ref_norm = ost.quantize_batch(keys)
    assert b.endswith(ref_pay.tobytes())
    mse = float(re.search(r"mse=(\S+)", out_c).group(1))
    assert abs(mse - float(np.mean(ref_norm.astype(np.float64) ** 2))) <= 1e-6 * mse


@pytest.mark.gpu
@pytest.mark.parametrize("square", [False, True])
def test_train_batch_bit_exact(square):
    """One trainer batch at D = 128 (vqkv_train_batch_host): loss sums and the projections' straight-through
    gradients equal the oracle's accumulate_loss (trainer.cpp:36-86)."""
    import ctypes as C

    from paper_2603_16435_b200 import _lib
    from paper_2603_16435_b200 import codebook as P

    rng = O.Rng(77)
    ost = rng.stack(4, 256, 128, O.KEY)
    pst = P.CodebookStack.from_arrays([ost.entries(s) for s in range(4)], [ost.projection(s) for s in range(4)], 0)
    x = O.generate(O.ROPE_ROTATED_KEYS, 128, 300, 8, 5)
    sums_ref, g_ref = O.train_batch(ost, x, beta=0.25, gamma=1.0, square_commitment=square)
    sums = np.zeros(3 + 4, np.float64)
    g = np.zeros((4, 128, 128), np.float32)
    _lib.call("vqkv_train_batch_host", pst.device.h, x.ctypes.data, 300, C.c_float(0.25), C.c_float(1.0), int(square),
              g.ctypes.data, sums.ctypes.data_as(C.POINTER(C.c_double)))
    assert np.array_equal(g, g_ref)
    assert np.allclose(sums, sums_ref, rtol=1e-12, atol=0)
