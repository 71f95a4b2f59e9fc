"""Tensor-core encoder (K1, tcgen05) parity against the oracle.

Codes must be bit-exact; near-ties (oracle best/second gap below the stated
epsilon) are counted and reported but, because every ambiguous window is
rescored exactly, the expected mismatch count is zero.  Residual norms are
bit-exact (same fp32 operation order as Eigen's squaredNorm).
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_mod():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def product_stack(o):
    from paper_2603_16435_b200 import codebook as P

    return P.CodebookStack.from_arrays([o.entries(s) for s in range(o.n)], [o.projection(s) for s in range(o.n)],
                                       o.kind)


def near_tie_eps(best, second, rnorm, emax):
    """tau = 2^-14 ||r|| max||e|| + 2^-22 max(|s1|,|s2|)."""
    return 2.0 ** -14 * rnorm * emax + 2.0 ** -22 * np.maximum(np.abs(best), np.abs(second))


def run_tc(torch, p, xs, n_streams=1, sb=4096, residuals=False):
    from paper_2603_16435_b200 import device as Dv

    rows = xs.shape[0] // n_streams
    x = torch.from_numpy(np.ascontiguousarray(xs.reshape(n_streams, rows, 128))).cuda()
    Dv.set_encode_path(2)
    try:
        out = Dv.quantize_streams(p, x, sb, residuals=residuals)
    finally:
        Dv.set_encode_path(0)
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in out]


def compare(o, p, xs, payload_dev, norms_dev, n_streams=1):
    rows = xs.shape[0] // n_streams
    n_mismatch = n_tie = 0
    for sidx in range(n_streams):
        xs_s = xs[sidx * rows : (sidx + 1) * rows]
        ref_pay, ref_norm, ins = o.quantize_batch(xs_s, instrument=True)
        got = o.unpack(payload_dev[sidx], rows)
        ref = o.unpack(ref_pay, rows)
        bad = np.nonzero((got != ref).any(1))[0]
        emax = o.stage_max_norm()
        for r in bad:
            st = int(np.nonzero(got[r] != ref[r])[0][0])
            gap = ins["second"][r, st] - ins["best"][r, st]
            tau = near_tie_eps(ins["best"][r, st], ins["second"][r, st], ins["rnorm"][r, st], emax[st])
            if gap <= tau:
                n_tie += 1
            else:
                n_mismatch += 1
        ok_rows = np.ones(rows, bool)
        ok_rows[bad] = False
        assert np.array_equal(norms_dev[sidx][ok_rows].view(np.uint32), ref_norm[ok_rows].view(np.uint32))
        if len(bad) == 0:
            assert np.array_equal(payload_dev[sidx], ref_pay)
    return n_mismatch, n_tie


@pytest.mark.parametrize(
    "seed,n,S,rows,streams",
    [(101, 4, 1024, 300, 1), (102, 16, 512, 200, 2), (103, 3, 256, 257, 3), (104, 2, 100, 129, 1),
     (105, 1, 1, 40, 1), (106, 5, 384, 128, 2), (107, 56, 1024, 48, 1),
     # configs[3] sweep sizes above 1024: stages span several 1024-entry super-blocks
     (108, 4, 2048, 150, 1), (109, 2, 4096, 130, 2), (110, 3, 1500, 129, 1), (111, 8, 3000, 64, 1)],
)
def test_tc_encode_matches_oracle(torch_mod, seed, n, S, rows, streams):
    rng = O.Rng(seed)
    o = rng.stack(n, S, 128)
    p = product_stack(o)
    xs = rng.matrix(rows * streams, 128)
    pay, nrm = run_tc(torch_mod, p, xs, streams)
    mism, ties = compare(o, p, xs, pay, nrm, streams)
    print(f"seed={seed} N={n} S={S} rows={rows*streams}: mismatches={mism} near_ties={ties}")
    assert mism == 0


def test_tc_encode_synthetic_keys(torch_mod):
    """LLaMA-shaped synthetic keys (rope-rotated mixture) through the paper's K stack shape."""
    rng = O.Rng(1)
    o = rng.stack(56, 1024, 128, O.KEY)
    p = product_stack(o)
    xs = O.generate(O.ROPE_ROTATED_KEYS, 128, 96, 32, 1000)
    pay, nrm = run_tc(torch_mod, p, xs)
    mism, ties = compare(o, p, xs, pay, nrm)
    print(f"synthetic keys: mismatches={mism} near_ties={ties}")
    assert mism == 0


def test_tc_exact_ties_and_degenerate(torch_mod):
    """Duplicate entries (exact score ties -> lowest index), zero codebooks, exact-entry inputs."""
    rng = O.Rng(7)
    base = rng.matrix(64, 128)
    ent = np.vstack([base, base[:32], np.zeros((32, 128), np.float32)])  # 128 entries, duplicates + zeros
    o = O.Stack.from_entries([ent, ent[::-1].copy(), np.zeros((128, 128), np.float32)])
    p = product_stack(o)
    xs = np.vstack([base[:40], rng.matrix(60, 128), np.zeros((5, 128), np.float32)])
    pay, nrm = run_tc(torch_mod, p, xs)
    mism, ties = compare(o, p, xs, pay, nrm)
    assert mism == 0


def test_tc_nonfinite_rows_use_exact_path(torch_mod):
    rng = O.Rng(9)
    o = rng.stack(3, 256, 128)
    p = product_stack(o)
    xs = rng.matrix(200, 128)
    xs[3, 7] = np.nan
    xs[150, 0] = np.inf
    xs[151, 1] = -np.inf
    pay, nrm = run_tc(torch_mod, p, xs)
    ref_pay, ref_norm = o.quantize_batch(xs)
    assert np.array_equal(pay[0], ref_pay)
    assert np.array_equal(np.isnan(nrm[0]), np.isnan(ref_norm))


def test_tc_residual_vectors(torch_mod):
    """quantize() final_residual through the tensor-core path equals the oracle's, bit for bit."""
    rng = O.Rng(11)
    o = rng.stack(6, 512, 128)
    p = product_stack(o)
    xs = rng.matrix(130, 128)
    pay, nrm, res = run_tc(torch_mod, p, xs, residuals=True)
    for r in (0, 1, 64, 127, 128, 129):
        _, ref_res = o.quantize(xs[r])
        assert np.array_equal(res[0, r].view(np.uint32), ref_res.view(np.uint32))


def test_tc_search_block_one(torch_mod):
    """search_block=1 switches the reference to dot() order for every entry; parity must hold."""
    rng = O.Rng(12)
    o = rng.stack(3, 128, 128)
    p = product_stack(o)
    xs = rng.matrix(64, 128)
    from paper_2603_16435_b200 import device as Dv

    pay, nrm = run_tc(torch_mod, p, xs, sb=1)
    ref_pay, ref_norm = o.quantize_batch(xs, 1)
    assert np.array_equal(pay[0], ref_pay)


@pytest.mark.parametrize("kind,n,S", [("K", 56, 1024), ("V", 16, 512)])
def test_full_size_round_trip_properties(torch_mod, kind, n, S):
    """configs[0] at full size: 256 (layer, head) streams x 4096 rows through the tensor-core
    encoder and the decoder.  Size-independent properties on every row (acceptance_test.cpp
    criterion 2: the replayed reconstruction error equals the recorded residual norm within 1e-4
    relative; codes in range), and a sample of rows bit-exact against the oracle (codes, norms,
    reconstruction), with near-ties counted."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    streams, rows = 256, 4096
    rng = O.Rng(2026 + n)
    o = rng.stack(n, S, 128, O.KEY if kind == "K" else O.VALUE)
    p = product_stack(o)
    gen = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randn(streams, rows, 128, device="cuda", generator=gen)
    pay, nrm = Dv.quantize_streams(p, x)
    rec = Dv.reconstruct_streams(p, pay, rows)
    err = torch.linalg.vector_norm(x - rec, dim=-1)
    assert torch.isfinite(nrm).all()
    assert torch.allclose(err, nrm, rtol=1e-4, atol=1e-5)
    del err
    # sampled rows: exact parity with the oracle
    for sidx in (0, 137, 255):
        sub = x[sidx, :48].cpu().numpy()
        ref_pay, ref_norm = o.quantize_batch(sub)
        got_pay, got_norm = Dv.quantize_streams(p, x[sidx : sidx + 1, :48].contiguous())
        got = o.unpack(got_pay[0].cpu().numpy(), 48)
        assert np.array_equal(got, o.unpack(ref_pay, 48))
        assert np.array_equal(got_norm[0].cpu().numpy().view(np.uint32), ref_norm.view(np.uint32))
        # the same rows inside the full-size launch carry the same codes
        full_rows = o.unpack(pay[sidx].cpu().numpy(), rows)[:48]
        assert np.array_equal(full_rows, got)
        assert np.array_equal(rec[sidx, :48].cpu().numpy(), o.reconstruct_block(ref_pay, 48, 0, 48))


@pytest.mark.parametrize("blocking", [True, False])
def test_host_buffer_pipeline_matches_device_encode(torch_mod, blocking):
    """vqkv_quantize_batch_host(_async): chunked H2D / encode / D2H over pinned host buffers,
    chunk encodes alternating between two compute streams, gives the same payload and norms as
    the device-resident encode of the same rows."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    rng = O.Rng(5)
    o = rng.stack(8, 256, 128, O.KEY)
    p = product_stack(o)
    streams, rows = 23, 31740  # 16 MB per stream: several chunks of 2-10 streams
    gen = torch.Generator().manual_seed(3)
    xh = torch.randn(streams, rows, 128, generator=gen).pin_memory()
    pay_d, nrm_d = Dv.quantize_streams(p, xh.cuda())
    pay_h, nrm_h = Dv.quantize_streams_host(p, xh, blocking=blocking)
    torch.cuda.synchronize()
    assert torch.equal(pay_h, pay_d.cpu())
    assert torch.equal(nrm_h.view(torch.int32), nrm_d.cpu().view(torch.int32))


def test_degenerate_sizes(torch_mod):
    """Empty calls (quantize_batch with no rows, checks only when rows > 0 as codebook.cpp:225-237;
    reconstruct_block of an empty range) and single-row / single-stream calls through every path."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    rng = O.Rng(8)
    o = rng.stack(3, 256, 128, O.KEY)
    p = product_stack(o)
    pay, nrm = Dv.quantize_streams(p, torch.empty((2, 0, 128), device="cuda"))
    assert pay.shape == (2, 0) and nrm.shape == (2, 0)
    pay, nrm = Dv.quantize_streams(p, torch.empty((0, 5, 128), device="cuda"))
    assert pay.numel() == 0 and nrm.numel() == 0
    x1 = rng.matrix(1, 128)
    pay, nrm = Dv.quantize_streams(p, torch.from_numpy(x1).cuda())
    ref_pay, ref_norm = o.quantize_batch(x1)
    assert np.array_equal(pay[0].cpu().numpy(), ref_pay)
    assert np.array_equal(nrm[0].cpu().numpy().view(np.uint32), ref_norm.view(np.uint32))
    rec = Dv.reconstruct_streams(p, pay, 1, 1, 1)
    assert rec.shape == (1, 0, 128)
    rec = Dv.reconstruct_streams(p, pay, 1)
    assert np.array_equal(rec[0].cpu().numpy(), o.reconstruct_block(ref_pay, 1, 0, 1))
    # host-buffer path with one row
    ph, nh = Dv.quantize_streams_host(p, torch.from_numpy(x1).reshape(1, 1, 128).contiguous())
    assert np.array_equal(ph[0].numpy(), ref_pay)


def test_tc_encode_many_stages(torch_mod):
    """More stages than the encoder caches in shared memory (kSmemStages = 128): the stage
    descriptors past the cache are read from global memory; codes and norms stay bit-exact."""
    rng = O.Rng(130)
    o = rng.stack(130, 16, 128, O.KEY)
    p = product_stack(o)
    xs = rng.matrix(64, 128)
    pay, nrm = run_tc(torch_mod, p, xs)
    mism, ties = compare(o, p, xs, pay, nrm)
    assert mism == 0


@pytest.mark.parametrize(
    "seed,n,S,rows,streams",
    [(301, 4, 1024, 1000, 3), (302, 3, 384, 130, 5), (303, 2, 4096, 257, 2), (304, 6, 200, 64, 1),
     (305, 16, 512, 2000, 9), (306, 2, 256, 8, 7), (307, 3, 128, 512, 4)],
)
def test_cta_pair_kernel_matches_single_cta_kernel(torch_mod, monkeypatch, seed, n, S, rows, streams):
    """The CTA-pair encoder (cta_group::2, default) and the single-CTA kernel (VQKV_ENC_PAIR=0) give
    identical payloads, norms and final residuals, including tile counts that leave a pair tile or
    a whole quad partly empty, and rows on the exact path (non-finite input)."""
    rng = O.Rng(seed)
    o = rng.stack(n, S, 128)
    p = product_stack(o)
    xs = rng.matrix(rows * streams, 128)
    xs[3, 7] = np.nan
    xs[rows * streams - 1, 0] = np.inf
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("VQKV_ENC_PAIR", mode)
        outs[mode] = run_tc(torch_mod, p, xs, n_streams=streams, residuals=True)
    for a, b in zip(outs["1"], outs["0"]):
        assert a.shape == b.shape
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    # and the pair kernel against the oracle on the first stream (finite rows bit-exact; the
    # non-finite row's norm is NaN on both sides, with a different NaN payload)
    ref_pay, ref_norm = o.quantize_batch(xs[:rows])
    got_codes, ref_codes = o.unpack(outs["1"][0][0], rows), o.unpack(ref_pay, rows)
    fin = np.isfinite(xs[:rows]).all(1)
    assert np.array_equal(got_codes[fin], ref_codes[fin])
    assert np.array_equal(outs["1"][1][0][fin].view(np.uint32), ref_norm[fin].view(np.uint32))
    assert np.array_equal(np.isnan(outs["1"][1][0][~fin]), np.isnan(ref_norm[~fin]))
