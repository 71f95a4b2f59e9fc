"""GPU parity tests: the CUDA path (through the C-ABI) against the CPU oracle.

Bar: bit-exact for codebooks, codes (modulo counted near-ties on the tensor-
core path), residual norms and reconstructions; attention within the stated
bf16 tolerance  max|o - o_ref| <= 2^-7 * max(1, max|o_ref|).
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ATT_TOL = 2.0 ** -7


def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def product_stack(ostack, device=0):
    from paper_2603_16435_b200 import codebook as P

    ents = [ostack.entries(s) for s in range(ostack.n)]
    projs = [ostack.projection(s) for s in range(ostack.n)]
    return P.CodebookStack.from_arrays(ents, projs, ostack.kind, device)


@pytest.fixture(scope="module")
def torch_mod():
    return torch_cuda()


@pytest.mark.parametrize("seed,n,S,D", [(1, 2, 16, 8), (2, 3, 33, 5), (3, 1, 1, 1), (4, 4, 256, 128), (5, 2, 7, 3)])
def test_stack_refresh_bit_exact(torch_mod, seed, n, S, D):
    """codebook.cpp:30-39 computed on the device == oracle restatement, bit for bit."""
    o = O.Rng(seed).stack(n, S, D)
    p = product_stack(o)
    for s in range(n):
        e, q = p.device.effective(s)
        assert np.array_equal(e.view(np.uint32), o.effective(s).view(np.uint32))
        assert np.array_equal(q.view(np.uint32), o.sqnorm(s).view(np.uint32))


@pytest.mark.parametrize("seed,n,S,D,rows", [(11, 3, 16, 8, 50), (12, 5, 300, 7, 33), (13, 2, 1024, 128, 300),
                                              (14, 1, 1, 4, 5), (15, 8, 256, 128, 130),
                                              # D = 128 with <= 32 stages (next-row code prefetch kernel),
                                              # exactly 32, and 40 (general kernel)
                                              (16, 16, 512, 128, 700), (17, 32, 100, 128, 90),
                                              (18, 40, 64, 128, 77)])
def test_reconstruct_block_bit_exact(torch_mod, seed, n, S, D, rows):
    """codebook.cpp:239-250 on random codes; every partition concatenates identically."""
    from paper_2603_16435_b200 import codebook as P

    rng = O.Rng(seed)
    o = rng.stack(n, S, D)
    p = product_stack(o)
    codes = np.array([[rng() % S for _ in range(n)] for _ in range(rows)], np.uint32)
    payload = o.pack(codes)
    ref = o.reconstruct_block(payload, rows, 0, rows)
    cm = P.CodeMatrix.from_payload(o.sizes, payload, rows)
    got = P.reconstruct_block(p, cm, 0, rows)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    b = 0
    while b < rows:
        e = min(rows, b + 1 + (b % 7))
        assert np.array_equal(P.reconstruct_block(p, cm, b, e), ref[b:e])
        b = e


def test_reconstruct_errors(torch_mod):
    """codebook.cpp:241-244 (range) and :216-219 (InvalidCode on foreign payloads)."""
    from paper_2603_16435_b200 import codebook as P
    from paper_2603_16435_b200 import errors as E

    o = O.Rng(21).stack(2, 5, 4)  # 3-bit fields can hold 5..7
    p = product_stack(o)
    cm = P.CodeMatrix.from_payload([5, 5], np.array([0xFF, 0x00], np.uint8), 1)  # code 7 in stage 0
    with pytest.raises(E.InvalidCode):
        P.reconstruct_block(p, cm, 0, 1)
    good = P.CodeMatrix([5, 5])
    good.append([1, 2])
    with pytest.raises(E.InvalidInput):
        P.reconstruct_block(p, good, 0, 2)
    with pytest.raises(E.InvalidInput):
        P.reconstruct_block(p, good, 1, 0)
    assert P.reconstruct_block(p, good, 1, 1).shape == (0, 4)
    # D = 128, few stages: the invalid code in the third row is reported, its neighbours decode
    o2 = O.Rng(22).stack(3, 5, 128)
    p2 = product_stack(o2)
    bad = P.CodeMatrix.from_payload([5, 5, 5], np.array([0x00, 0x00, 0x00, 0x00, 0xFF, 0x01], np.uint8), 5)
    with pytest.raises(E.InvalidCode):
        P.reconstruct_block(p2, bad, 0, 5)


def _encode_cases():
    return [(31, 3, 16, 8, 64, 4096), (32, 2, 33, 5, 40, 1), (33, 2, 33, 5, 40, 7), (34, 4, 300, 9, 70, 4096),
            (35, 2, 1024, 128, 64, 4096), (36, 1, 1, 3, 10, 4096), (37, 8, 256, 64, 100, 32)]


@pytest.mark.parametrize("seed,n,S,D,rows,sb", _encode_cases())
def test_encode_exact_path_bit_exact(torch_mod, seed, n, S, D, rows, sb):
    """quantize_batch (codebook.cpp:225-237) on the exact SIMT path: payload bytes and norms identical."""
    from paper_2603_16435_b200 import codebook as P
    from paper_2603_16435_b200 import device as Dv

    rng = O.Rng(seed)
    o = rng.stack(n, S, D)
    xs = rng.matrix(rows, D)
    ref_pay, ref_norm = o.quantize_batch(xs, sb)
    p = product_stack(o)
    Dv.set_encode_path(1)
    try:
        r = P.quantize_batch(p, xs, sb)
    finally:
        Dv.set_encode_path(0)
    assert np.array_equal(r.codes.payload(), ref_pay)
    assert np.array_equal(r.residual_norms.view(np.uint32), ref_norm.view(np.uint32))


def test_encode_kats_on_device(torch_mod):
    """codebook_test.cpp KATs through the product API."""
    from paper_2603_16435_b200 import codebook as P

    E = lambda r: np.array(r, np.float32)
    st = P.CodebookStack.from_arrays([E([[0, 0], [1, 0], [0, 1]])])
    nr = P.nearest_entry(st.stages[0], [0.9, 0.1])
    assert nr.index == 1 and nr.distance == pytest.approx(0.14142136, rel=1e-4)
    st = P.CodebookStack.from_arrays([E([[1, 0], [1, 0]])])
    assert P.nearest_entry(st.stages[0], [1.0, 0.0]).index == 0
    st = P.CodebookStack.from_arrays([E([[0.5, 0.25], [-1, 2], [3, 1]])])
    q = P.quantize(st, [-1.0, 2.0])
    assert q.codes == [1] and np.linalg.norm(q.final_residual) == 0.0
    st = P.CodebookStack.from_arrays([E([[1, 0], [0, 1]]), E([[0, 0.5], [0.5, 0]])])
    q = P.quantize(st, [1.2, 0.4])
    assert q.codes == [0, 0]
    assert q.final_residual[0] == pytest.approx(0.2, rel=1e-6) and q.final_residual[1] == pytest.approx(-0.1, rel=1e-6)
    rec = P.reconstruct(st, q.codes)
    assert rec[0] == pytest.approx(1.0) and rec[1] == pytest.approx(0.5)
    st = P.CodebookStack.from_arrays([E([[1, 0], [0, 1], [1, 1], [2, 2]])])
    r = P.quantize_batch(st, E([[1, 1], [2, 2], [0, 1]]))
    assert [r.codes.row(i) for i in range(3)] == [[2], [3], [1]] and r.residual_norms.max() == 0.0
    st = P.CodebookStack.from_arrays([np.zeros((3, 4), np.float32), np.zeros((2, 4), np.float32)])
    x = O.Rng(5).matrix(1, 4)[0]
    q = P.quantize(st, x)
    assert q.codes == [0, 0] and np.allclose(q.final_residual, x)
    r = P.quantize_batch(st, np.zeros((0, 4), np.float32))
    assert r.codes.rows() == 0 and r.residual_norms.size == 0


def test_encode_nonfinite_rows_follow_reference(torch_mod):
    """quantize has no finiteness check (codebook.cpp:194-206): NaN rows pick index 0 every stage."""
    from paper_2603_16435_b200 import codebook as P

    rng = O.Rng(41)
    o = rng.stack(3, 64, 128)
    xs = rng.matrix(8, 128)
    xs[2, 5] = np.nan
    xs[5, 0] = np.inf
    ref_pay, ref_norm = o.quantize_batch(xs)
    p = product_stack(o)
    r = P.quantize_batch(p, xs)
    assert np.array_equal(r.codes.payload(), ref_pay)
    assert np.array_equal(np.isnan(r.residual_norms), np.isnan(ref_norm))
    fin = ~np.isnan(ref_norm)
    assert np.array_equal(r.residual_norms[fin], ref_norm[fin])


def test_attention_generic_vs_oracle(torch_mod):
    """attend (attention.cpp:26-69) over init | compressed | local, GQA group 4."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    rng = O.Rng(51)
    ks = rng.stack(3, 16, 8, O.KEY)
    vs = rng.stack(2, 8, 8, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    n_pairs, G, n_init, n_comp, n_local = 3, 4, 2, 37, 5
    init_k = rng.matrix(n_pairs * n_init, 8).reshape(n_pairs, n_init, 8)
    init_v = rng.matrix(n_pairs * n_init, 8).reshape(n_pairs, n_init, 8)
    loc_k = rng.matrix(n_pairs * n_local, 8).reshape(n_pairs, n_local, 8)
    loc_v = rng.matrix(n_pairs * n_local, 8).reshape(n_pairs, n_local, 8)
    kcodes = [ks.pack(np.array([[rng() % 16 for _ in range(3)] for _ in range(n_comp)], np.uint32)) for _ in range(n_pairs)]
    vcodes = [vs.pack(np.array([[rng() % 8 for _ in range(2)] for _ in range(n_comp)], np.uint32)) for _ in range(n_pairs)]
    q = rng.matrix(n_pairs * G, 8).reshape(n_pairs, G, 8)
    dev = "cuda:0"
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    out, lse = Dv.attend_decode(pk, pv, t(q), t(np.stack(kcodes)), t(np.stack(vcodes)), n_comp,
                                t(init_k), t(init_v), t(loc_k), t(loc_v))
    out = out.cpu().numpy()
    lse = lse.cpu().numpy()
    for pi in range(n_pairs):
        for g in range(G):
            ref, ref_lse = O.attend_segments(ks, vs, init_k[pi], init_v[pi], kcodes[pi], vcodes[pi], n_comp,
                                             loc_k[pi], loc_v[pi], q[pi, g])
            tol = ATT_TOL * max(1.0, np.abs(ref).max())
            assert np.abs(out[pi, g] - ref).max() <= tol
            assert abs(lse[pi, g] - ref_lse) <= 1e-3 * max(1.0, abs(ref_lse))


def test_lse_combine_matches_monolithic(torch_mod):
    """Sequence split into 4 shards + LSE merge == attention over the whole sequence."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    rng = O.Rng(61)
    ks = rng.stack(2, 32, 16, O.KEY)
    vs = rng.stack(2, 32, 16, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    n_comp, parts, G = 200, 4, 4
    codes_k = np.array([[rng() % 32 for _ in range(2)] for _ in range(n_comp)], np.uint32)
    codes_v = np.array([[rng() % 32 for _ in range(2)] for _ in range(n_comp)], np.uint32)
    q = rng.matrix(G, 16).reshape(1, G, 16)
    dev = "cuda:0"
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    full, full_lse = Dv.attend_decode(pk, pv, t(q), t(ks.pack(codes_k)[None]), t(vs.pack(codes_v)[None]), n_comp)
    outs, lses = [], []
    per = n_comp // parts
    for i in range(parts):
        sl = slice(i * per, (i + 1) * per)
        o_, l_ = Dv.attend_decode(pk, pv, t(q), t(ks.pack(codes_k[sl])[None]), t(vs.pack(codes_v[sl])[None]), per)
        outs.append(o_.reshape(G, 16))
        lses.append(l_.reshape(G))
    mo, ml = Dv.lse_combine(torch.stack(outs).contiguous(), torch.stack(lses).contiguous())
    assert torch.allclose(mo, full.reshape(G, 16), atol=1e-5, rtol=1e-4)
    assert torch.allclose(ml, full_lse.reshape(G), atol=1e-5, rtol=1e-5)


@pytest.mark.parametrize("nk,sk,nv,sv,n_pairs,n_init,n_comp,n_local",
                         [(6, 256, 4, 128, 3, 4, 9000, 40), (56, 1024, 16, 512, 2, 4, 3000, 17), (56, 1024, 16, 512, 1, 3, 8300, 5), (3, 64, 2, 64, 2, 0, 100, 0),
                          (4, 128, 4, 128, 1, 2, 0, 33),
                          # > 18 value stages: value-code windows read one at a time; 8192-token split edge
                          (8, 512, 24, 64, 2, 4, 8192, 8), (9, 1024, 40, 32, 1, 1, 8193, 2),
                          # more pairs than SMs: CTA token ranges span several pairs (several segments per CTA)
                          (4, 128, 4, 128, 200, 2, 600, 3), (56, 1024, 16, 512, 300, 1, 10, 2),
                          # pairs spanning 3-5 CTAs (one chunk each): accumulators handed over across CTA
                          # boundaries, including chains through single-segment middle CTAs
                          (4, 128, 4, 128, 1, 2, 40000, 3), (8, 256, 4, 128, 3, 1, 20000, 2)])
def test_attention_lut_path_vs_oracle(torch_mod, nk, sk, nv, sv, n_pairs, n_init, n_comp, n_local):
    """LUT/histogram fast path (D=128, G=4) against the oracle's attend over the same segments."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    rng = O.Rng(nk * 1000 + sk)
    ks = rng.stack(nk, sk, 128, O.KEY)
    vs = rng.stack(nv, sv, 128, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    G = 4
    mk = lambda n: rng.matrix(max(n_pairs * n, 1), 128)[: n_pairs * n].reshape(n_pairs, n, 128)
    init_k, init_v, loc_k, loc_v = mk(n_init), mk(n_init), mk(n_local), mk(n_local)
    g = np.random.default_rng(nk)
    kc = np.stack([ks.pack(g.integers(0, sk, (n_comp, nk)).astype(np.uint32)) for _ in range(n_pairs)])
    vc = np.stack([vs.pack(g.integers(0, sv, (n_comp, nv)).astype(np.uint32)) for _ in range(n_pairs)])
    q = rng.matrix(n_pairs * G, 128).reshape(n_pairs, G, 128)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out, lse = Dv.attend_decode(pk, pv, t(q), t(kc) if n_comp else None, t(vc) if n_comp else None, n_comp,
                                t(init_k) if n_init else None, t(init_v) if n_init else None,
                                t(loc_k) if n_local else None, t(loc_v) if n_local else None)
    out, lse = out.cpu().numpy(), lse.cpu().numpy()
    worst = 0.0
    for pi in range(n_pairs):
        for gg in range(G):
            ref, ref_lse = O.attend_segments(ks, vs, init_k[pi], init_v[pi], kc[pi] if n_comp else b"", vc[pi] if n_comp else b"",
                                             n_comp, loc_k[pi], loc_v[pi], q[pi, gg])
            err = np.abs(out[pi, gg] - ref).max() / max(1.0, np.abs(ref).max())
            worst = max(worst, err)
            assert abs(lse[pi, gg] - ref_lse) <= 1e-3 * max(1.0, abs(ref_lse))
    print(f"worst scaled attention error {worst:.2e} (tolerance {ATT_TOL:.2e})")
    assert worst <= ATT_TOL


@pytest.mark.parametrize("G", [1, 2, 3, 6, 8, 13])
def test_attention_other_group_sizes_use_lut_path(torch_mod, monkeypatch, G):
    """Group sizes other than 4 run through the LUT path in groups of 4 heads (the last one padded):
    same results as the oracle and as the generic kernel (VQKV_ATTEND_PATH=1)."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    nk, sk, nv, sv, n_pairs, n_init, n_comp, n_local = 56, 1024, 16, 512, 3, 4, 2500, 9
    rng = O.Rng(900 + G)
    ks = rng.stack(nk, sk, 128, O.KEY)
    vs = rng.stack(nv, sv, 128, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    mk = lambda n: rng.matrix(n_pairs * n, 128).reshape(n_pairs, n, 128)
    init_k, init_v, loc_k, loc_v = mk(n_init), mk(n_init), mk(n_local), mk(n_local)
    g = np.random.default_rng(G)
    kc = np.stack([ks.pack(g.integers(0, sk, (n_comp, nk)).astype(np.uint32)) for _ in range(n_pairs)])
    vc = np.stack([vs.pack(g.integers(0, sv, (n_comp, nv)).astype(np.uint32)) for _ in range(n_pairs)])
    q = rng.matrix(n_pairs * G, 128).reshape(n_pairs, G, 128)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    run = lambda: [x.cpu().numpy() for x in Dv.attend_decode(pk, pv, t(q), t(kc), t(vc), n_comp, t(init_k), t(init_v),
                                                             t(loc_k), t(loc_v))]
    out, lse = run()
    monkeypatch.setenv("VQKV_ATTEND_PATH", "1")
    out_g, lse_g = run()
    monkeypatch.delenv("VQKV_ATTEND_PATH")
    assert out.shape == (n_pairs, G, 128) and lse.shape == (n_pairs, G)
    assert np.abs(out - out_g).max() <= ATT_TOL * max(1.0, np.abs(out_g).max())
    assert np.abs(lse - lse_g).max() <= 1e-3 * max(1.0, np.abs(lse_g).max())
    for pi in range(n_pairs):
        for gg in (0, G - 1):
            ref, ref_lse = O.attend_segments(ks, vs, init_k[pi], init_v[pi], kc[pi], vc[pi], n_comp, loc_k[pi], loc_v[pi],
                                             q[pi, gg])
            assert np.abs(out[pi, gg] - ref).max() <= ATT_TOL * max(1.0, np.abs(ref).max())
            assert abs(lse[pi, gg] - ref_lse) <= 1e-3 * max(1.0, abs(ref_lse))


def gm_records_np(ks, codes, cap, t0=0):
    """The attention record layout (include/vqkv_c.h) built in numpy from unpacked codes: per
    group of 8 key stages, token t's 80-bit record holds in field k the code of stage
    8g + ((t & 7) ^ k); planes of cap u64 (bits 0-63) then cap u16 (bits 64-79)."""
    n_rows, n = codes.shape
    ng = (n + 7) // 8
    out = np.zeros(ng * cap * 10, np.uint8)
    t = np.arange(t0, t0 + n_rows)
    for g in range(ng):
        lo = np.zeros(n_rows, np.uint64)
        hi = np.zeros(n_rows, np.uint64)
        for k in range(8):
            s = 8 * g + ((t & 7) ^ k)
            z = np.where(s < n, codes[np.arange(n_rows), np.minimum(s, n - 1)], 0).astype(np.uint64)
            b = 10 * k
            if b + 10 <= 64:
                lo |= z << np.uint64(b)
            elif b >= 64:
                hi |= z << np.uint64(b - 64)
            else:
                lo |= (z << np.uint64(b)) & np.uint64(0xFFFFFFFFFFFFFFFF)
                hi |= z >> np.uint64(64 - b)
        seg = out[g * cap * 10:(g + 1) * cap * 10]
        seg[: 8 * cap].view(np.uint64)[t0:t0 + n_rows] = lo
        seg[8 * cap: 10 * cap].view(np.uint16)[t0:t0 + n_rows] = hi.astype(np.uint16)
    return out


@pytest.mark.parametrize("nk,sk,nv,sv,n_pairs,n_init,n_comp,n_local",
                         [(56, 1024, 16, 512, 2, 4, 3000, 17), (56, 1024, 16, 512, 1, 3, 8300, 5),
                          (6, 256, 4, 128, 3, 4, 9000, 40), (5, 1000, 3, 64, 2, 0, 700, 3), (1, 9, 1, 4, 1, 1, 40, 0)])
def test_attention_group_major_keys(torch_mod, monkeypatch, nk, sk, nv, sv, n_pairs, n_init, n_comp, n_local):
    """Attention records: the transcoder writes the documented records and inverts them back to
    the CodeMatrix payload byte for byte; attention over them equals attention over the CodeMatrix
    rows bit for bit (the rows are transcoded to the same records) and matches the oracle."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    rng = O.Rng(nk * 7 + sk)
    ks = rng.stack(nk, sk, 128, O.KEY)
    vs = rng.stack(nv, sv, 128, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    G = 4
    mk = lambda n: rng.matrix(max(n_pairs * n, 1), 128)[: n_pairs * n].reshape(n_pairs, n, 128)
    init_k, init_v, loc_k, loc_v = mk(n_init), mk(n_init), mk(n_local), mk(n_local)
    g = np.random.default_rng(nk + 1)
    kcodes = [g.integers(0, sk, (n_comp, nk)).astype(np.uint32) for _ in range(n_pairs)]
    kc = np.stack([ks.pack(c) for c in kcodes])
    vc = np.stack([vs.pack(g.integers(0, sv, (n_comp, nv)).astype(np.uint32)) for _ in range(n_pairs)])
    q = rng.matrix(n_pairs * G, 128).reshape(n_pairs, G, 128)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    cap = -(-n_comp // 16) * 16 + 32  # spare capacity
    gm = Dv.keycodes_to_gm(pk, t(kc), n_comp, cap=cap, gm=torch.zeros((n_pairs, Dv.keycodes_gm_bytes(pk, cap)),
                                                                     dtype=torch.uint8, device="cuda"))
    gm_h = gm.cpu().numpy()
    for pi in range(n_pairs):
        assert np.array_equal(gm_h[pi], gm_records_np(ks, kcodes[pi], cap))
    back = Dv.keycodes_from_gm(pk, gm, cap, n_comp).cpu().numpy()
    assert np.array_equal(back, kc)
    seg = lambda a, n: t(a) if n else None
    args = (seg(init_k, n_init), seg(init_v, n_init), seg(loc_k, n_local), seg(loc_v, n_local))
    o_rows, l_rows = Dv.attend_decode(pk, pv, t(q), t(kc), t(vc), n_comp, *args)
    o_gm, l_gm = Dv.attend_decode(pk, pv, t(q), gm, t(vc), n_comp, *args, kcodes_gm_cap=cap)
    assert torch.equal(l_rows, l_gm) and torch.equal(o_rows, o_gm)
    out = o_gm.cpu().numpy()
    for pi in range(n_pairs):
        for gg in range(G):
            ref, _ = O.attend_segments(ks, vs, init_k[pi], init_v[pi], kc[pi], vc[pi], n_comp, loc_k[pi], loc_v[pi],
                                       q[pi, gg])
            assert np.abs(out[pi, gg] - ref).max() <= ATT_TOL * max(1.0, np.abs(ref).max())


def test_group_major_errors(torch_mod):
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv
    from paper_2603_16435_b200.errors import InvalidInput

    rng = O.Rng(3)
    pk = product_stack(rng.stack(4, 2048, 128, O.KEY))  # > 1024 entries: no group-major layout
    assert Dv.keycodes_gm_bytes(pk, 64) == 0
    ks = rng.stack(4, 64, 128, O.KEY)
    pk, pv = product_stack(ks), product_stack(rng.stack(2, 64, 128, O.VALUE))
    assert Dv.keycodes_gm_bytes(pk, 24) == 0  # cap not a multiple of 16
    kc = torch.zeros((1, ks.payload_bytes(100)), dtype=torch.uint8, device="cuda")
    vc = torch.zeros((1, 100), dtype=torch.uint8, device="cuda")
    gm = Dv.keycodes_to_gm(pk, kc, 100, cap=112)
    q = torch.randn(1, 4, 128, device="cuda")
    with pytest.raises(InvalidInput):
        Dv.attend_decode(pk, pv, q, gm, vc, 100, kcodes_gm_cap=96)  # cap < n_comp
    with pytest.raises(InvalidInput):
        Dv.keycodes_to_gm(pk, kc, 100, gm=gm, cap=112, dst_row=20)  # past the capacity


@pytest.mark.parametrize("qscale", [1.0, 1e-3, 40.0])
def test_attention_lut_tensor_core_vs_ffma(torch_mod, monkeypatch, qscale):
    """The tensor-core LUT GEMM (fp16 hi/lo split, default for D = 128) against the fp32 FFMA
    LUT kernel (VQKV_LUT_FFMA=1): same attention within fp32-level differences, and both
    within the stated tolerance of the oracle."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    nk, sk, nv, sv, n_pairs, n_comp = 56, 1024, 16, 512, 37, 3000  # 148 query rows: two row tiles
    rng = O.Rng(91)
    ks, vs = rng.stack(nk, sk, 128, O.KEY), rng.stack(nv, sv, 128, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    g = np.random.default_rng(9)
    kc = np.stack([ks.pack(g.integers(0, sk, (n_comp, nk)).astype(np.uint32)) for _ in range(n_pairs)])
    vc = np.stack([vs.pack(g.integers(0, sv, (n_comp, nv)).astype(np.uint32)) for _ in range(n_pairs)])
    q = (rng.matrix(n_pairs * 4, 128) * np.float32(qscale)).reshape(n_pairs, 4, 128)
    lk, lv = rng.matrix(n_pairs * 8, 128).reshape(n_pairs, 8, 128), rng.matrix(n_pairs * 8, 128).reshape(n_pairs, 8, 128)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("VQKV_LUT_FFMA", mode)
        res[mode] = Dv.attend_decode(pk, pv, t(q), t(kc), t(vc), n_comp, None, None, t(lk), t(lv))
    (o1, l1), (o2, l2) = res["1"], res["0"]
    assert torch.allclose(l1, l2, rtol=1e-5, atol=1e-5)
    assert torch.allclose(o1, o2, rtol=1e-4, atol=1e-4 * max(1.0, float(o1.abs().max())))
    out = o2.cpu().numpy()
    for pi in (0, n_pairs - 1):
        for gg in range(4):
            ref, _ = O.attend_segments(ks, vs, np.zeros((0, 128), np.float32), np.zeros((0, 128), np.float32), kc[pi],
                                       vc[pi], n_comp, lk[pi], lv[pi], q[pi, gg])
            assert np.abs(out[pi, gg] - ref).max() <= ATT_TOL * max(1.0, np.abs(ref).max())


def test_sequence_split_lut_path_matches_monolithic(torch_mod):
    """configs[4] on one GPU: the 8-rank sequence split of bench.py (sharding.sequence_shards:
    init rows on shard 0, local window on the last), each shard's (o, lse) from the group-major LUT
    path, merged by the library's LSE combine == attention over the whole sequence; then the same
    partials through sharding.gather_and_merge over a world-size-1 NCCL group."""
    torch = torch_mod
    import socket
    import torch.distributed as dist
    from paper_2603_16435_b200 import device as Dv, sharding

    nk, sk, nv, sv, world = 56, 1024, 16, 512, 8
    n_init, n_comp, n_local, heads = 4, 20000, 64, 2
    rng = O.Rng(123)
    ks, vs = rng.stack(nk, sk, 128, O.KEY), rng.stack(nv, sv, 128, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    g = np.random.default_rng(3)
    kcodes = [g.integers(0, sk, (n_comp, nk)).astype(np.uint32) for _ in range(heads)]
    vcodes = [g.integers(0, sv, (n_comp, nv)).astype(np.uint32) for _ in range(heads)]
    ik, iv = rng.matrix(heads * n_init, 128).reshape(heads, n_init, 128), rng.matrix(heads * n_init, 128).reshape(heads, n_init, 128)
    lk, lv = rng.matrix(heads * n_local, 128).reshape(heads, n_local, 128), rng.matrix(heads * n_local, 128).reshape(heads, n_local, 128)
    q = rng.matrix(heads * 4, 128).reshape(heads, 4, 128)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()

    def attend(c0, c1, init, local):
        nc = c1 - c0
        kc = t(np.stack([ks.pack(kcodes[h][c0:c1]) for h in range(heads)]))
        vc = t(np.stack([vs.pack(vcodes[h][c0:c1]) for h in range(heads)]))
        cap = -(-max(nc, 1) // Dv.GM_ALIGN) * Dv.GM_ALIGN
        kg = Dv.keycodes_to_gm(pk, kc, nc, cap=cap)
        seg = lambda a, on: t(a) if on else None
        return Dv.attend_decode(pk, pv, t(q), kg, vc, nc, seg(ik, init), seg(iv, init), seg(lk, local), seg(lv, local),
                                kcodes_gm_cap=cap)

    full_o, full_l = attend(0, n_comp, True, True)
    parts = [attend(sh.comp[0], sh.comp[1], sh.init[1] > 0, sh.local[1] > 0)
             for sh in sharding.sequence_shards(n_init, n_comp, n_local, world)]
    o_all = torch.stack([p[0].reshape(-1, 128) for p in parts]).contiguous()
    l_all = torch.stack([p[1].reshape(-1) for p in parts]).contiguous()
    mo, ml = Dv.lse_combine(o_all, l_all)
    assert torch.allclose(mo, full_o.reshape(-1, 128), rtol=1e-4, atol=1e-4 * max(1.0, float(full_o.abs().max())))
    assert torch.allclose(ml, full_l.reshape(-1), rtol=1e-5, atol=1e-5)

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        o1, l1 = sharding.gather_and_merge(parts[3][0], parts[3][1])
        r1, rl1 = Dv.lse_combine(parts[3][0].reshape(1, -1, 128).contiguous(), parts[3][1].reshape(1, -1).contiguous())
        assert torch.allclose(o1.reshape(-1, 128), r1, rtol=1e-6, atol=1e-6)
        assert torch.allclose(l1.reshape(-1), rl1, rtol=1e-6, atol=1e-6)
    finally:
        dist.destroy_process_group()

    # the C-ABI exchange step a C++ host calls (vqkv_lse_allgather_combine over an ncclCommInitAll
    # communicator): world size 1 here, so the merge of the gathered partial is the partial itself
    comms = sharding.NcclComms([0])
    try:
        o2, l2 = sharding.nccl_gather_and_merge(comms.comm(0), parts[5][0].reshape(-1, 128), parts[5][1].reshape(-1))
        torch.cuda.synchronize()
        r2, rl2 = Dv.lse_combine(parts[5][0].reshape(1, -1, 128).contiguous(), parts[5][1].reshape(1, -1).contiguous())
        assert torch.allclose(o2, r2, rtol=1e-6, atol=1e-6)
        assert torch.allclose(l2, rl2, rtol=1e-6, atol=1e-6)
    finally:
        comms.close()


def test_attention_lut_large_entries_fall_back_to_ffma(torch_mod):
    """Key entries beyond the fp16 range (|e| >= 2^15) take the FFMA LUT build instead of the
    tensor-core GEMM; the result matches the oracle within the tolerance."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    nk, sk, nv, sv, n_comp = 4, 256, 2, 64, 500
    g = np.random.default_rng(17)
    kent = [(g.standard_normal((sk, 128)) * (4e4 if s == 1 else 1.0)).astype(np.float32) for s in range(nk)]
    vent = [g.standard_normal((sv, 128)).astype(np.float32) for _ in range(nv)]
    ks, vs = O.Stack.from_entries(kent, kind=O.KEY), O.Stack.from_entries(vent, kind=O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    kc = ks.pack(g.integers(0, sk, (n_comp, nk)).astype(np.uint32))
    vc = vs.pack(g.integers(0, sv, (n_comp, nv)).astype(np.uint32))
    q = (g.standard_normal((1, 4, 128)) * 1e-5).astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out, _ = Dv.attend_decode(pk, pv, t(q), t(kc[None]), t(vc[None]), n_comp)
    out = out.cpu().numpy()
    z = np.zeros((0, 128), np.float32)
    for gg in range(4):
        ref, _ = O.attend_segments(ks, vs, z, z, kc, vc, n_comp, z, z, q[0, gg])
        assert np.abs(out[0, gg] - ref).max() <= ATT_TOL * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("gap", [13.5, 20.0, 26.0])
def test_attention_value_path_near_flat_tail(torch_mod, gap):
    """Adversarial for the value histograms: 8192 tokens whose weights sit `gap` nats below one
    dominant token (13.5: just under round 1's absolute 2^-19 cut; 26: deep in the tail), with
    values on the opposite side, so the tail's mass (8192 e^-gap of the top weight) moves the
    output by up to |v_a - v_b| times it.  The relative fixed point keeps every such token:
    within the tolerance of the oracle and of the closed form, whichever chunk the top token is in."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    D, n_tail = 128, 8192
    u = np.zeros(D, np.float32)
    u[0] = 1.0
    kent = np.zeros((16, D), np.float32)
    kent[0] = 30.0 * u
    kent[1] = (30.0 - gap) * u
    vent = np.zeros((16, D), np.float32)
    vent[0] = 1.0
    vent[1] = -1.0
    ks, vs = O.Stack.from_entries([kent], kind=O.KEY), O.Stack.from_entries([vent], kind=O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    q = np.tile((u * np.sqrt(D)).astype(np.float32), (1, 4, 1))  # scale * q . e = u . e
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    z = np.zeros((0, D), np.float32)
    for top in (n_tail, 0, 5000):  # the dominant token after, before and inside the tail
        codes = np.ones((n_tail + 1, 1), np.uint32)
        codes[top] = 0
        kc, vc = ks.pack(codes), vs.pack(codes)
        out, lse = Dv.attend_decode(pk, pv, t(q), t(kc[None]), t(vc[None]), n_tail + 1)
        out = out.cpu().numpy()
        w = n_tail * np.exp(-gap)
        exact = (1.0 - w) / (1.0 + w)
        ref, _ = O.attend_segments(ks, vs, z, z, kc, vc, n_tail + 1, z, z, q[0, 0])
        for g in range(4):
            assert np.abs(out[0, g] - ref).max() <= ATT_TOL * max(1.0, np.abs(ref).max())
            assert np.abs(out[0, g] - exact).max() <= 2.0 ** -16 + 1e-5
