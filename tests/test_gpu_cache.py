"""Device-resident batched CacheState (paper_2603_16435_b200/cache.py) against the oracle's
CacheState restatement (oracle/vqkv_oracle.cpp, kv_cache.cpp:41-204), one oracle cache per stream.

Bar: counts, code payloads, residual norms and view_block rows bit-exact; memory_report equal;
attention over the cache within the stated tolerance max|o - o_ref| <= 2^-7 * max(1, max|o_ref|).
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ATT_TOL = 2.0 ** -7


@pytest.fixture(scope="module")
def torch_mod():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def product_stack(ostack):
    from paper_2603_16435_b200 import codebook as P

    return P.CodebookStack.from_arrays([ostack.entries(s) for s in range(ostack.n)],
                                       [ostack.projection(s) for s in range(ostack.n)], ostack.kind, 0)


def check_state(torch, dc, refs, ks, vs, q, check_attention=True):
    S = dc.n_streams
    for r in refs:
        assert dc.counts() == r.counts()
    # code payloads and residual norms, per stream
    for which, st in ((0, ks), (1, vs)):
        pay, nrm = dc.codes(which)
        pay, nrm = pay.cpu().numpy(), nrm.cpu().numpy()
        for i, r in enumerate(refs):
            rp, rn = r.codes(which)
            assert np.array_equal(pay[i], rp)
            assert np.array_equal(nrm[i].view(np.uint32), rn.view(np.uint32))
    L = dc.total_len()
    k, v, ex = dc.view_block(0, L)
    k, v, ex = k.cpu().numpy(), v.cpu().numpy(), ex.numpy()
    for i, r in enumerate(refs):
        rk, rv, rex = r.view_block(0, L)
        assert np.array_equal(k[i].view(np.uint32), rk.view(np.uint32))
        assert np.array_equal(v[i].view(np.uint32), rv.view(np.uint32))
        assert np.array_equal(ex, rex)
    # an inner window crossing segment boundaries
    if L > 3:
        b, e = 1, L - 1
        k2, v2, ex2 = dc.view_block(b, e)
        assert np.array_equal(k2.cpu().numpy(), k[:, b:e]) and np.array_equal(ex2.numpy(), ex[b:e])
    rep = dc.memory_report()
    ref_rep = refs[0].memory_report()
    for key in ("raw_bytes_equivalent", "compressed_payload_bits", "codebook_overhead_bytes"):
        assert rep[key] == ref_rep[key], key
    assert abs(rep["effective_ratio"] - ref_rep["effective_ratio"]) < 1e-12
    if check_attention:
        out, lse = dc.attend(torch.from_numpy(q).cuda())
        out = out.cpu().numpy()
        for i, r in enumerate(refs):
            for g in range(q.shape[1]):
                ref = r.attend(q[i, g])
                assert np.abs(out[i, g] - ref).max() <= ATT_TOL * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("eager", [False, True])
@pytest.mark.parametrize("D,nk,sk,nv,sv", [(8, 3, 16, 2, 8), (128, 4, 64, 3, 32)])
def test_cache_lifecycle_vs_oracle(torch_mod, eager, D, nk, sk, nv, sv):
    """prefill -> decode steps with evictions, deferred/eager flushes -> every observable equal."""
    torch = torch_mod
    from paper_2603_16435_b200.cache import DeviceCacheState

    rng = O.Rng(7000 + D + int(eager))
    ks, vs = rng.stack(nk, sk, D, O.KEY), rng.stack(nv, sv, D, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    S, G, init_len, local_len, L0, steps = 3, 4, 2, 5, 13, 17
    refs = [O.Cache(ks, vs, init_len, local_len, eager) for _ in range(S)]
    dc = DeviceCacheState(pk, pv, S, init_len, local_len, eager)
    keys = rng.matrix(S * L0, D).reshape(S, L0, D)
    vals = rng.matrix(S * L0, D).reshape(S, L0, D)
    for i, r in enumerate(refs):
        r.prefill(keys[i], vals[i])
    dc.prefill(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda())
    q = rng.matrix(S * G, D).reshape(S, G, D)
    check_state(torch, dc, refs, ks, vs, q)
    for step in range(steps):
        k1, v1 = rng.matrix(S, D), rng.matrix(S, D)
        for i, r in enumerate(refs):
            r.append_token(k1[i], v1[i])
        dc.append_token(torch.from_numpy(k1).cuda(), torch.from_numpy(v1).cuda())
        if step % 4 == 3 or step == steps - 1:
            check_state(torch, dc, refs, ks, vs, q)
    assert dc.counts()["batched"] >= 1


def test_cache_short_prefill_and_no_prefill(torch_mod):
    """prefill shorter than init + local (nothing compressed); init_len == 0 allows appends first."""
    torch = torch_mod
    from paper_2603_16435_b200.cache import DeviceCacheState

    rng = O.Rng(7100)
    ks, vs = rng.stack(2, 16, 8, O.KEY), rng.stack(2, 16, 8, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    q = rng.matrix(2 * 4, 8).reshape(2, 4, 8)
    refs = [O.Cache(ks, vs, 4, 3, False) for _ in range(2)]
    dc = DeviceCacheState(pk, pv, 2, 4, 3)
    x = rng.matrix(2 * 5, 8).reshape(2, 5, 8)
    for i, r in enumerate(refs):
        r.prefill(x[i], x[i])
    dc.prefill(torch.from_numpy(x).cuda(), torch.from_numpy(x).cuda())
    check_state(torch, dc, refs, ks, vs, q)
    refs = [O.Cache(ks, vs, 0, 2, False) for _ in range(2)]
    dc = DeviceCacheState(pk, pv, 2, 0, 2)
    for _ in range(7):
        k1 = rng.matrix(2, 8)
        for i, r in enumerate(refs):
            r.append_token(k1[i], k1[i])
        dc.append_token(torch.from_numpy(k1).cuda(), torch.from_numpy(k1).cuda())
    check_state(torch, dc, refs, ks, vs, q)


def test_cache_errors(torch_mod):
    """Error kinds of kv_cache.cpp (InvalidState / InvalidInput)."""
    torch = torch_mod
    from paper_2603_16435_b200.cache import DeviceCacheState
    from paper_2603_16435_b200.errors import InvalidInput, InvalidState

    rng = O.Rng(7200)
    ks, vs = rng.stack(2, 16, 8, O.KEY), rng.stack(2, 16, 8, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    with pytest.raises(InvalidInput):
        DeviceCacheState(pk, pv, 2, 4, 0)
    dc = DeviceCacheState(pk, pv, 2, 4, 3)
    one = torch.zeros(2, 8, device="cuda")
    with pytest.raises(InvalidState):
        dc.append_token(one, one)
    with pytest.raises(InvalidState):
        dc.attend(torch.zeros(2, 4, 8, device="cuda"))
    with pytest.raises(InvalidInput):
        dc.prefill(torch.zeros(2, 0, 8, device="cuda"), torch.zeros(2, 0, 8, device="cuda"))
    with pytest.raises(InvalidInput):
        dc.prefill(torch.zeros(2, 3, 7, device="cuda"), torch.zeros(2, 3, 8, device="cuda"))
    dc.prefill(torch.zeros(2, 3, 8, device="cuda"), torch.zeros(2, 3, 8, device="cuda"))
    with pytest.raises(InvalidState):
        dc.prefill(torch.zeros(2, 3, 8, device="cuda"), torch.zeros(2, 3, 8, device="cuda"))
    with pytest.raises(InvalidInput):
        dc.view_block(2, 5)
    with pytest.raises(InvalidInput):
        dc.append_token(torch.zeros(3, 8, device="cuda"), torch.zeros(3, 8, device="cuda"))


def test_payload_append_bit_offsets(torch_mod):
    """vqkv_payload_append == CodeMatrix::append row by row, at every bit alignment."""
    torch = torch_mod
    from paper_2603_16435_b200 import _lib

    rng = O.Rng(7300)
    st = rng.stack(3, 5, 4, O.KEY)  # 3 bits x 3 stages = 9-bit rows
    codes = np.array([[rng() % 5 for _ in range(3)] for _ in range(40)], np.uint32)
    full = st.pack(codes)
    for cut in (0, 1, 7, 8, 13, 39):
        a, b = st.pack(codes[:cut]), st.pack(codes[cut:])
        dst = torch.zeros((2, len(full) + 3), dtype=torch.uint8, device="cuda")
        dst[:, : len(a)] = torch.from_numpy(np.frombuffer(bytes(a), np.uint8).copy()).cuda() if len(a) else 0
        src = torch.from_numpy(np.stack([np.frombuffer(bytes(b), np.uint8)] * 2).copy()).cuda()
        _lib.call("vqkv_payload_append", dst.data_ptr(), dst.stride(0), cut * 9, src.data_ptr(), src.stride(0),
                  (40 - cut) * 9, 2, torch.cuda.current_stream().cuda_stream)
        got = dst.cpu().numpy()
        for i in range(2):
            assert np.array_equal(got[i, : len(full)], np.frombuffer(bytes(full), np.uint8)), cut


@pytest.mark.parametrize("D,Q", [(8, 4), (128, 4), (8, 40), (128, 40)])
def test_cache_fidelity_vs_oracle(torch_mod, D, Q):
    """fidelity (attention.cpp:90-134): reconstruction MSE exact, attention-based fields within
    tolerance; any number of queries (Q = 40: ten groups of the kernels' G = 4)."""
    torch = torch_mod
    from paper_2603_16435_b200.cache import DeviceCacheState

    rng = O.Rng(7400 + D)
    ks, vs = rng.stack(3, 32, D, O.KEY), rng.stack(2, 16, D, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    S, L = 2, 40
    refs = [O.Cache(ks, vs, 3, 8, False) for _ in range(S)]
    dc = DeviceCacheState(pk, pv, S, 3, 8)
    keys = rng.matrix(S * L, D).reshape(S, L, D)
    vals = rng.matrix(S * L, D).reshape(S, L, D)
    for i, r in enumerate(refs):
        r.prefill(keys[i], vals[i])
    dc.prefill(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda())
    q = rng.matrix(S * Q, D).reshape(S, Q, D)
    rep = dc.fidelity(torch.from_numpy(keys).cuda(), torch.from_numpy(vals).cuda(), torch.from_numpy(q).cuda())
    for i, r in enumerate(refs):
        comp = np.stack([r.attend(q[i, j]) for j in range(Q)]).astype(np.float64)
        raw = np.stack([O.attend_raw(keys[i], vals[i], q[i, j]) for j in range(Q)]).astype(np.float64)
        ref_err = np.abs(comp - raw).max()
        cos = np.mean([(c @ w) / (np.linalg.norm(c) * np.linalg.norm(w)) for c, w in zip(comp, raw)])
        tol = ATT_TOL * max(1.0, np.abs(raw).max())
        assert abs(rep["output_max_abs_err"][i].item() - ref_err) <= 2 * tol
        assert abs(rep["output_mean_cosine"][i].item() - cos) <= 1e-3
        rk, rv, ex = r.view_block(0, L)
        mid = ~ex
        kmse = np.mean(np.sum((keys[i][mid].astype(np.float64) - rk[mid]) ** 2, axis=1))
        vmse = np.mean(np.sum((vals[i][mid].astype(np.float64) - rv[mid]) ** 2, axis=1))
        # the reference evaluates these in fp32 (MatrixF arithmetic): fp32-level agreement
        assert abs(rep["key_intermediate_mse"][i].item() - kmse) <= 1e-6 * max(1.0, kmse)
        assert abs(rep["value_intermediate_mse"][i].item() - vmse) <= 1e-6 * max(1.0, vmse)


def _vqks_from_oracle(r, ks, vs, init_len, local_len, eager, prefilled, kst_host, vst_host):
    """An independent restatement of CacheState::save_snapshot (kv_cache.cpp:206-245) built
    from the oracle cache's observable state -- the expected bytes for one stream."""
    import struct

    from paper_2603_16435_b200.codebook import stack_content_hash

    c = r.counts()
    L = c["total"]
    k, v, ex = r.view_block(0, L)
    ni, nc, npd = c["init"], c["compressed"], c["pending"]
    kp, kn = r.codes(0)
    vp, vn = r.codes(1)
    b = b"VQKS" + struct.pack("<IQQBBQII", 1, init_len, local_len, int(eager), int(prefilled), L, ks.dim, vs.dim)
    b += struct.pack("<QQQ", stack_content_hash(kst_host), stack_content_hash(vst_host), c["batched"])
    b += struct.pack("<Q", ni) + k[:ni].tobytes() + struct.pack("<Q", ni) + v[:ni].tobytes()
    for st, pay in ((ks, kp), (vs, vp)):
        b += struct.pack("<I", st.n) + b"".join(struct.pack("<I", x) for x in st.sizes) + struct.pack("<Q", nc)
        b += bytes(pay)
    b += kn.tobytes() + vn.tobytes()
    t0 = ni + nc
    for rows in (k[t0:t0 + npd], v[t0:t0 + npd], k[t0 + npd:], v[t0 + npd:]):
        b += struct.pack("<Q", len(rows)) + rows.tobytes()
    return b


def test_cache_vqks_snapshots(torch_mod, tmp_path):
    """VQKS snapshots (kv_cache.cpp:206-312): bytes equal an independent restatement from the
    oracle's state; loading them back gives an identical batched cache."""
    import io

    torch = torch_mod
    from paper_2603_16435_b200.cache import DeviceCacheState
    from paper_2603_16435_b200.errors import InvalidInput

    rng = O.Rng(7500)
    ks, vs = rng.stack(3, 16, 8, O.KEY), rng.stack(2, 8, 8, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    S, init_len, local_len = 2, 2, 4
    refs = [O.Cache(ks, vs, init_len, local_len, False) for _ in range(S)]
    dc = DeviceCacheState(pk, pv, S, init_len, local_len)
    x = rng.matrix(S * 11, 8).reshape(S, 11, 8)
    y = rng.matrix(S * 11, 8).reshape(S, 11, 8)
    for i, r in enumerate(refs):
        r.prefill(x[i], y[i])
    dc.prefill(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    for _ in range(6):  # leaves pending rows and one flush behind
        k1, v1 = rng.matrix(S, 8), rng.matrix(S, 8)
        for i, r in enumerate(refs):
            r.append_token(k1[i], v1[i])
        dc.append_token(torch.from_numpy(k1).cuda(), torch.from_numpy(v1).cuda())
    paths = []
    for i, r in enumerate(refs):
        buf = io.BytesIO()
        dc.save_snapshot(i, buf)
        assert buf.getvalue() == _vqks_from_oracle(r, ks, vs, init_len, local_len, False, True, pk, pv)
        p = str(tmp_path / f"s{i}.vqks")
        dc.save_snapshot(i, p)
        paths.append(p)
    back = DeviceCacheState.load_snapshots(paths, pk, pv)
    q = rng.matrix(S * 4, 8).reshape(S, 4, 8)
    check_state(torch, back, refs, ks, vs, q)
    other = product_stack(rng.stack(3, 16, 8, O.KEY))
    with pytest.raises(InvalidInput):
        DeviceCacheState.load_snapshots(paths, other, pv)


def test_cache_snapshot_rejects_out_of_range_codes(torch_mod):
    """A VQKS file whose codes exceed their stage size (S = 12 -> 4-bit fields) is rejected with
    InvalidCode at load, as the reference rejects it when decoding (codebook.cpp:212-217), and a
    file written for other stage sizes with InvalidInput."""
    import io
    import struct

    from paper_2603_16435_b200.cache import DeviceCacheState
    from paper_2603_16435_b200.errors import InvalidCode

    rng = O.Rng(7777)
    ks, vs = rng.stack(2, 12, 8, O.KEY), rng.stack(2, 12, 8, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    r = O.Cache(ks, vs, 2, 4, False)
    r.prefill(rng.matrix(20, 8), rng.matrix(20, 8))
    good = _vqks_from_oracle(r, ks, vs, 2, 4, False, True, pk, pv)
    DeviceCacheState.load_snapshots([io.BytesIO(good)], pk, pv)  # loads
    # the key CodeMatrix payload starts after the header, the init rows and its own header
    c = r.counts()
    off = 4 + struct.calcsize("<IQQBBQII") + 24 + 2 * (8 + 4 * 8 * c["init"]) + 4 + 4 * 2 + 8
    bad = bytearray(good)
    bad[off] = 0xFF  # row 0: both 4-bit fields = 15 >= 12
    with pytest.raises(InvalidCode):
        DeviceCacheState.load_snapshots([io.BytesIO(bytes(bad))], pk, pv)


def test_cache_attention_records_only(torch_mod, tmp_path):
    """The key codes live only as attention records (no CodeMatrix copy on the device): kept in
    step through prefill, flushes and capacity growth (planes copied) and snapshot loads; the
    CodeMatrix rows rebuilt from them equal the rows-layout cache's payload byte for byte, and
    attention over them equals attention over the rows-layout cache bit for bit and the oracle."""
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv
    from paper_2603_16435_b200.cache import DeviceCacheState

    rng = O.Rng(7700)
    ks, vs = rng.stack(5, 256, 128, O.KEY), rng.stack(3, 64, 128, O.VALUE)
    pk, pv = product_stack(ks), product_stack(vs)
    S, init_len, local_len, L0 = 2, 4, 64, 2000
    dc = DeviceCacheState(pk, pv, S, init_len, local_len)
    rows = DeviceCacheState(pk, pv, S, init_len, local_len, attn_layout="rows")
    assert dc.attn_layout == "group_major" and dc.kpay is None and rows.kgm is None
    ref = O.Cache(ks, vs, init_len, local_len, False)
    x = rng.matrix(S * L0, 128).reshape(S, L0, 128)
    y = rng.matrix(S * L0, 128).reshape(S, L0, 128)
    for c in (dc, rows):
        c.prefill(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    ref.prefill(x[0], y[0])
    q = rng.matrix(S * 4, 128).reshape(S, 4, 128)
    qt = torch.from_numpy(q).cuda()

    def check(c):
        assert torch.equal(c.codes(0)[0], rows.codes(0)[0])
        o, l = c.attend(qt)
        o2, l2 = rows.attend(qt)
        assert torch.equal(l, l2) and torch.equal(o, o2)
        for g in range(4):
            r = ref.attend(q[0, g])
            assert np.abs(o[0, g].cpu().numpy() - r).max() <= ATT_TOL * max(1.0, np.abs(r).max())
        rp, _ = ref.codes(0)
        assert np.array_equal(c.codes(0)[0][0].cpu().numpy(), rp)

    check(dc)
    cap0 = dc.cap_rows
    for _ in range(3 * local_len):  # flushes, then growth past the first capacity
        k1, v1 = rng.matrix(S, 128), rng.matrix(S, 128)
        ref.append_token(k1[0], v1[0])
        for c in (dc, rows):
            c.append_token(torch.from_numpy(k1).cuda(), torch.from_numpy(v1).cuda())
    assert dc.cap_rows > cap0 and dc.counts()["batched"] >= 2
    check(dc)
    # 5 key stages = 1 group of 8: 10 B per token, + 3 x 6-bit value fields
    assert dc.memory_report()["device_code_bytes"] == dc.n_comp * 10 + pv_bytes(dc)
    paths = []
    for i in range(S):
        paths.append(str(tmp_path / f"s{i}.vqks"))
        dc.save_snapshot(i, paths[-1])
    back = DeviceCacheState.load_snapshots(paths, pk, pv)
    assert back.attn_layout == "group_major" and back.kpay is None
    check(back)


def pv_bytes(c):
    return c.vd.payload_bytes(c.n_comp)
