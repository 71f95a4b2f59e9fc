"""Pins the CPU oracle against the reference's own known-answer tests.

Each test ports a doctest case from /root/reference/proj/tests (file:line in
the docstring) and runs it on the oracle restatement.  No GPU needed.
"""
import numpy as np
import pytest

from oracle import oracle as O


def E(rows):
    return np.array(rows, np.float32)


# ---------------- codebook_test.cpp ----------------

def test_nearest_entry_picks_closest():
    """codebook_test.cpp:35-42"""
    st = O.Stack.from_entries([E([[0, 0], [1, 0], [0, 1]])])
    idx, dist = st.nearest_entry(0, [0.9, 0.1])
    assert idx == 1
    assert dist == pytest.approx(0.14142136, rel=1e-4)


def test_nearest_entry_exact_match_zero_distance():
    """codebook_test.cpp:44-50"""
    st = O.Stack.from_entries([E([[0.3, -1.2], [2.0, 0.5], [-0.7, 0.9]])])
    idx, dist = st.nearest_entry(0, st.effective(0)[2])
    assert idx == 2 and dist == 0.0


def test_nearest_entry_tie_lowest_index():
    """codebook_test.cpp:52-57"""
    st = O.Stack.from_entries([E([[1, 0], [1, 0]])])
    assert st.nearest_entry(0, [1.0, 0.0])[0] == 0


def test_nearest_entry_dim_mismatch():
    """codebook_test.cpp:59-64"""
    st = O.Stack.from_entries([E([[1, 0], [0, 1]])])
    with pytest.raises(O.OracleError) as e:
        st.nearest_entry(0, np.zeros(3, np.float32))
    assert e.value.code == O.INVALID_INPUT


def test_duplicating_entry_never_changes_index():
    """codebook_test.cpp:66-79"""
    rng = O.Rng(11)
    st = rng.stack(1, 16, 6)
    ent, proj = st.entries(0), st.projection(0)
    for _ in range(50):
        x = rng.matrix(1, 6)[0]
        base = st.nearest_entry(0, x)[0]
        dup = O.Stack.from_entries([np.vstack([ent, ent[base : base + 1]])], [proj])
        assert dup.nearest_entry(0, x)[0] == base


def test_quantize_representable_zero_residual():
    """codebook_test.cpp:81-88"""
    st = O.Stack.from_entries([E([[0.5, 0.25], [-1, 2], [3, 1]])])
    codes, res = st.quantize([-1.0, 2.0])
    assert list(codes) == [1]
    assert np.linalg.norm(res) == 0.0


def test_quantize_two_stage_walk():
    """codebook_test.cpp:90-103"""
    st = O.Stack.from_entries([E([[1, 0], [0, 1]]), E([[0, 0.5], [0.5, 0]])])
    codes, res = st.quantize([1.2, 0.4])
    assert list(codes) == [0, 0]
    assert res[0] == pytest.approx(0.2, rel=1e-6)
    assert res[1] == pytest.approx(-0.1, rel=1e-6)
    rec = st.reconstruct(codes)
    assert rec[0] == pytest.approx(1.0) and rec[1] == pytest.approx(0.5)


def test_all_zero_codebooks_noop():
    """codebook_test.cpp:105-112"""
    st = O.Stack.from_entries([np.zeros((3, 4), np.float32), np.zeros((2, 4), np.float32)])
    x = O.Rng(5).matrix(1, 4)[0]
    codes, res = st.quantize(x)
    assert list(codes) == [0, 0]
    np.testing.assert_allclose(res, x)


def test_residual_identity_random():
    """codebook_test.cpp:114-128"""
    rng = O.Rng(42)
    for _ in range(100):
        n = 1 + rng() % 4
        d = 2 + rng() % 15
        st = rng.stack(n, 8, d)
        x = rng.matrix(1, d)[0]
        codes, res = st.quantize(x)
        rt = st.reconstruct(codes) + res
        assert np.linalg.norm(rt - x) <= 1e-5 * max(1e-6, np.linalg.norm(x))
        err = np.linalg.norm(x - st.reconstruct(codes))
        assert np.linalg.norm(res) == pytest.approx(err, rel=1e-5)


def test_single_stage_reconstruct_effective():
    """codebook_test.cpp:130-136"""
    st = O.Rng(3).stack(1, 5, 7)
    for k in range(5):
        np.testing.assert_allclose(st.reconstruct([k]), st.effective(0)[k], rtol=1e-6)


def test_reconstruct_rejects_out_of_range():
    """codebook_test.cpp:138-143"""
    st = O.Rng(4).stack(2, 4, 3)
    for codes in ([0, 4], [0]):
        with pytest.raises(O.OracleError) as e:
            st.reconstruct(codes)
        assert e.value.code == O.INVALID_CODE


def test_quantize_batch_empty():
    """codebook_test.cpp:145-151"""
    st = O.Rng(6).stack(2, 4, 3)
    payload, norms = st.quantize_batch(np.zeros((0, 3), np.float32))
    assert payload.size == 0 and norms.size == 0


def test_quantize_batch_exact_entries():
    """codebook_test.cpp:153-162"""
    st = O.Stack.from_entries([E([[1, 0], [0, 1], [1, 1], [2, 2]])])
    payload, norms = st.quantize_batch(E([[1, 1], [2, 2], [0, 1]]))
    assert st.unpack(payload, 3).tolist() == [[2], [3], [1]]
    assert norms.max() == 0.0


def test_quantize_batch_matches_per_row():
    """codebook_test.cpp:164-174"""
    rng = O.Rng(7)
    st = rng.stack(3, 4, 8)
    xs = rng.matrix(16, 8)
    payload, norms = st.quantize_batch(xs)
    codes = st.unpack(payload, 16)
    for r in range(16):
        c, res = st.quantize(xs[r])
        assert list(codes[r]) == list(c)
        # codebook_test.cpp:172 asserts exact equality with the per-row norm
        n_ref = st.quantize_batch(xs[r : r + 1])[1][0]
        assert norms[r] == n_ref


def test_search_block_invariance():
    """codebook_test.cpp:176-186"""
    rng = O.Rng(8)
    st = rng.stack(2, 33, 5)
    xs = rng.matrix(10, 5)
    p0, n0 = st.quantize_batch(xs, 4096)
    for blk in (1, 3, 7, 32, 33):
        p1, n1 = st.quantize_batch(xs, blk)
        assert np.array_equal(p0, p1)
        assert np.array_equal(n0, n1)


def test_reconstruct_block_partitions():
    """codebook_test.cpp:188-210"""
    rng = O.Rng(9)
    st = rng.stack(3, 6, 4)
    xs = rng.matrix(10, 4)
    payload, _ = st.quantize_batch(xs)
    full = st.reconstruct_block(payload, 10, 0, 10)
    for blk in range(1, 5):
        b = 0
        while b < 10:
            e = min(10, b + blk)
            assert np.array_equal(st.reconstruct_block(payload, 10, b, e), full[b:e])
            b = e
    assert st.reconstruct_block(payload, 10, 4, 4).shape[0] == 0
    for b, e in ((4, 11), (5, 4)):
        with pytest.raises(O.OracleError) as ex:
            st.reconstruct_block(payload, 10, b, e)
        assert ex.value.code == O.INVALID_INPUT


def test_code_matrix_roundtrip():
    """codebook_test.cpp:212-235"""
    rng = O.Rng(10)
    for _ in range(20):
        n = 1 + rng() % 5
        sizes = [1 + rng() % 300 for _ in range(n)]
        rows = rng() % 40
        truth = np.array([[rng() % s for s in sizes] for _ in range(rows)], np.uint32).reshape(rows, n)
        payload = O.pack_codes(sizes, truth)
        assert np.array_equal(O.unpack_codes(sizes, payload, rows), truth)


def test_code_matrix_append_straddle():
    """codebook_test.cpp:237-249"""
    rng = O.Rng(12)
    truth = []
    for r in range(30):
        truth.append([rng() % 5, rng() % 3])
        p = O.pack_codes([5, 3], np.array(truth, np.uint32))
        assert np.array_equal(O.unpack_codes([5, 3], p, r + 1), np.array(truth))


def test_code_matrix_rejects_bad_append():
    """codebook_test.cpp:251-255"""
    with pytest.raises(O.OracleError) as e:
        O.pack_codes([4, 4], np.array([[4, 0]], np.uint32))
    assert e.value.code == O.INVALID_CODE


def test_stack_save_load_roundtrip(tmp_path):
    """codebook_test.cpp:257-273"""
    st = O.Rng(13).stack(3, 9, 6, O.VALUE)
    p = str(tmp_path / "s.rsvq")
    st.save(p)
    ld = O.Stack.load(p)
    assert ld.n == 3 and ld.kind == O.VALUE
    for i in range(3):
        assert np.array_equal(ld.entries(i), st.entries(i))
        assert np.array_equal(ld.projection(i), st.projection(i))
        np.testing.assert_allclose(ld.effective(i), st.effective(i), rtol=1e-6)
    assert ld.hash() == st.hash()


def test_stack_loader_byte_offsets():
    """codebook_test.cpp:275-296"""
    st = O.Rng(14).stack(1, 4, 3)
    b = bytearray(st.to_bytes())
    bad = bytes(b"X") + bytes(b[1:])
    with pytest.raises(O.OracleError) as e:
        O.Stack.from_bytes(bad)
    assert e.value.code == O.FORMAT_ERROR and e.value.offset == 0
    with pytest.raises(O.OracleError) as e:
        O.Stack.from_bytes(bytes(b[:-5]))
    assert e.value.code == O.FORMAT_ERROR


# ---------------- attention_test.cpp ----------------

class Fx:
    """attention_test.cpp:15-29 Fixture (rng 202, 3x16 stacks at D=8)."""

    def __init__(self):
        self.rng = O.Rng(202)
        self.ks = self.rng.stack(3, 16, 8, O.KEY)
        self.vs = self.rng.stack(3, 16, 8, O.VALUE)

    def filled(self, n, init=2, local=6):
        c = O.Cache(self.ks, self.vs, init, local)
        self.keys = self.rng.matrix(n, 8)
        self.values = self.rng.matrix(n, 8)
        c.prefill(self.keys, self.values)
        return c


def test_attend_single_token():
    """attention_test.cpp:33-38"""
    f = Fx()
    c = f.filled(1)
    q = f.rng.matrix(1, 8)[0]
    np.testing.assert_allclose(c.attend(q), f.values[0], rtol=1e-6)


def test_attend_block_rows_invariant():
    """attention_test.cpp:40-52"""
    f = Fx()
    c = f.filled(40)
    for _ in range(5):
        q = f.rng.matrix(1, 8)[0]
        whole = c.attend(q, 40)
        for rows in (1, 7, 13):
            assert np.abs(c.attend(q, rows) - whole).max() < 1e-6


def test_attend_streaming_matches_monolithic():
    """attention_test.cpp:54-65"""
    f = Fx()
    c = f.filled(32)
    for _ in range(5):
        q = f.rng.matrix(1, 8)[0]
        k, v, _ = c.view_block(0, 32)
        assert np.abs(c.attend(q, 5) - O.attend_raw(k, v, q)).max() < 1e-6


def test_attend_all_raw():
    """attention_test.cpp:67-75"""
    f = Fx()
    c = f.filled(8, 2, 6)
    assert c.counts()["compressed"] == 0
    q = f.rng.matrix(1, 8)[0]
    assert np.abs(c.attend(q, 3) - O.attend_raw(f.keys, f.values, q)).max() < 1e-6


def test_attend_weights_sum_to_one():
    """attention_test.cpp:77-98"""
    f = Fx()
    c = O.Cache(f.ks, f.vs, 2, 6)
    ks = f.rng.matrix(20, 8)
    c.prefill(ks, np.ones((20, 8), np.float32))
    q = f.rng.matrix(1, 8)[0]
    k, v, _ = c.view_block(0, 20)
    assert np.abs(c.attend(q, 4) - O.attend_raw(k, v, q)).max() < 1e-6
    raw = O.Cache(f.ks, f.vs, 4, 16)
    raw.prefill(ks, np.ones((20, 8), np.float32))
    assert np.abs(raw.attend(q, 4) - 1.0).max() < 1e-6


def test_attend_validates():
    """attention_test.cpp:100-109"""
    f = Fx()
    empty = O.Cache(f.ks, f.vs, 2, 6)
    with pytest.raises(O.OracleError) as e:
        empty.attend(np.zeros(8, np.float32))
    assert e.value.code == O.INVALID_STATE
    c = f.filled(10)
    with pytest.raises(O.OracleError) as e:
        c.attend(np.zeros(7, np.float32))
    assert e.value.code == O.INVALID_INPUT
    with pytest.raises(O.OracleError) as e:
        c.attend(np.zeros(8, np.float32), 0)
    assert e.value.code == O.INVALID_INPUT


def test_attend_stats():
    """attention_test.cpp:111-121"""
    f = Fx()
    c = f.filled(40, 2, 6)
    assert c.counts()["compressed"] == 32
    _, st = c.attend(f.rng.matrix(1, 8)[0], 4, stats=True)
    assert st["reconstructed_rows"] == 32
    assert 0 < st["peak_reconstructed_scalars"] <= 4 * 16


# ---------------- kv_cache_test.cpp ----------------

class KFx:
    """kv_cache_test.cpp:18-26 (rng 101, K 2x8 D=6, V 2x8 D=4)."""

    def __init__(self):
        self.rng = O.Rng(101)
        self.ks = self.rng.stack(2, 8, 6, O.KEY)
        self.vs = self.rng.stack(2, 8, 4, O.VALUE)

    def make(self, init, local, eager=False):
        return O.Cache(self.ks, self.vs, init, local, eager)


def test_prefill_segments():
    """kv_cache_test.cpp:30-54"""
    f = KFx()
    c = f.make(4, 8)
    c.prefill(f.rng.matrix(12, 6), f.rng.matrix(12, 4))
    assert c.counts() == dict(init=4, compressed=0, pending=0, local=8, total=12, batched=0)
    c = f.make(4, 16)
    c.prefill(f.rng.matrix(64, 6), f.rng.matrix(64, 4))
    cnt = c.counts()
    assert (cnt["init"], cnt["compressed"], cnt["local"], cnt["total"]) == (4, 44, 16, 64)
    c = f.make(4, 8)
    c.prefill(f.rng.matrix(1, 6), f.rng.matrix(1, 4))
    cnt = c.counts()
    assert (cnt["init"], cnt["compressed"], cnt["local"]) == (1, 0, 0)


def test_prefill_errors():
    """kv_cache_test.cpp:56-65"""
    f = KFx()
    c = f.make(2, 4)
    c.prefill(f.rng.matrix(8, 6), f.rng.matrix(8, 4))
    with pytest.raises(O.OracleError) as e:
        c.prefill(f.rng.matrix(8, 6), f.rng.matrix(8, 4))
    assert e.value.code == O.INVALID_STATE
    fresh = f.make(2, 4)
    with pytest.raises(O.OracleError) as e:
        fresh.prefill(np.zeros((0, 6), np.float32), np.zeros((0, 4), np.float32))
    assert e.value.code == O.INVALID_INPUT
    with pytest.raises(O.OracleError) as e:
        fresh.prefill(f.rng.matrix(4, 5), f.rng.matrix(4, 4))
    assert e.value.code == O.INVALID_INPUT


def test_appends_defer_quantization():
    """kv_cache_test.cpp:67-87"""
    f = KFx()
    c = f.make(2, 8)
    c.prefill(f.rng.matrix(10, 6), f.rng.matrix(10, 4))
    assert c.counts()["batched"] == 0
    c.append_token(f.rng.matrix(1, 6)[0], f.rng.matrix(1, 4)[0])
    assert c.counts()["batched"] == 0 and c.counts()["pending"] == 1
    for _ in range(7):
        c.append_token(f.rng.matrix(1, 6)[0], f.rng.matrix(1, 4)[0])
    cnt = c.counts()
    assert (cnt["batched"], cnt["pending"], cnt["compressed"], cnt["total"]) == (1, 0, 8, 18)


def test_append_requires_prefill():
    """kv_cache_test.cpp:89-96"""
    f = KFx()
    c = f.make(2, 4)
    with pytest.raises(O.OracleError) as e:
        c.append_token(np.zeros(6, np.float32), np.zeros(4, np.float32))
    assert e.value.code == O.INVALID_STATE
    z = f.make(0, 4)
    z.append_token(np.zeros(6, np.float32), np.zeros(4, np.float32))
    assert z.counts()["total"] == 1
    with pytest.raises(O.OracleError) as e:
        z.append_token(np.zeros(5, np.float32), np.zeros(4, np.float32))
    assert e.value.code == O.INVALID_INPUT


def test_eager_equals_deferred():
    """kv_cache_test.cpp:98-116"""
    f = KFx()
    keys, values = f.rng.matrix(40, 6), f.rng.matrix(40, 4)
    d, e = f.make(2, 6), f.make(2, 6, True)
    d.prefill(keys[:10], values[:10])
    e.prefill(keys[:10], values[:10])
    for t in range(10, 40):
        d.append_token(keys[t], values[t])
        e.append_token(keys[t], values[t])
    common = min(d.counts()["compressed"], e.counts()["compressed"])
    assert common > 0
    dk = f.ks.unpack(d.codes(0)[0], d.counts()["compressed"])[:common]
    ek = f.ks.unpack(e.codes(0)[0], e.counts()["compressed"])[:common]
    assert np.array_equal(dk, ek)
    assert e.counts()["pending"] == 0


def test_replay_view_block():
    """kv_cache_test.cpp:118-144"""
    f = KFx()
    keys, values = f.rng.matrix(60, 6), f.rng.matrix(60, 4)
    c = f.make(3, 7)
    c.prefill(keys[:20], values[:20])
    for t in range(20, 60):
        c.append_token(keys[t], values[t])
        cnt = c.counts()
        assert cnt["total"] == t + 1 == cnt["init"] + cnt["compressed"] + cnt["pending"] + cnt["local"]
    k, v, ex = c.view_block(0, 60)
    _, kn = c.codes(0)
    for t in range(60):
        if ex[t]:
            assert np.array_equal(k[t], keys[t]) and np.array_equal(v[t], values[t])
        else:
            err = np.linalg.norm(k[t] - keys[t])
            assert err == pytest.approx(kn[t - c.counts()["init"]], rel=1e-4)


def test_view_block_boundaries():
    """kv_cache_test.cpp:146-172"""
    f = KFx()
    keys, values = f.rng.matrix(30, 6), f.rng.matrix(30, 4)
    c = f.make(3, 7)
    c.prefill(keys, values)
    assert c.counts()["compressed"] == 20
    k, v, ex = c.view_block(25, 30)
    assert ex.all() and np.array_equal(k, keys[25:])
    _, _, ex = c.view_block(1, 6)
    assert ex[0] and ex[1] and not ex[2] and not ex[4]
    assert c.view_block(5, 5)[0].shape[0] == 0
    for b, e in ((5, 31), (9, 5)):
        with pytest.raises(O.OracleError) as er:
            c.view_block(b, e)
        assert er.value.code == O.INVALID_INPUT


def test_memory_report():
    """kv_cache_test.cpp:174-201"""
    f = KFx()
    c = f.make(2, 4)
    r = c.memory_report()
    assert r["raw_bytes_equivalent"] == 0 and r["compressed_payload_bits"] == 0 and r["effective_ratio"] == 0
    c = f.make(2, 8)
    c.prefill(f.rng.matrix(10, 6), f.rng.matrix(10, 4))
    r = c.memory_report()
    assert r["compressed_payload_bits"] == 0 and r["raw_bytes_equivalent"] == 10 * 10 * 2
    c = f.make(2, 4)
    c.prefill(f.rng.matrix(16, 6), f.rng.matrix(16, 4))
    r = c.memory_report()
    assert r["compressed_payload_bits"] == 10 * 2 * 3 * 2
    assert r["effective_ratio"] == pytest.approx(1 - 120.0 / (10 * 10 * 16.0), rel=1e-12)
    assert r["codebook_overhead_bytes"] > 0


# ---------------- acceptance_test.cpp criteria 2-5 ----------------

def test_acceptance_2_residual_identity():
    """acceptance_test.cpp:79-102 (10000 vectors, seed 1001)"""
    rng = O.Rng(1001)
    checked = ok = 0
    while checked < 10000:
        n = 1 + rng() % 8
        s = 2 + rng() % 255
        d = 1 + rng() % 64
        st = rng.stack(n, s, d)
        i = 0
        while i < 100 and checked < 10000:
            x = rng.matrix(1, d)[0]
            codes, res = st.quantize(x)
            rel = np.linalg.norm((st.reconstruct(codes) + res - x).astype(np.float32)) / max(
                1e-12, np.linalg.norm(x)
            )
            ok += rel <= 1e-5
            i += 1
            checked += 1
    assert ok == checked


def test_acceptance_3_batch_equivalence():
    """acceptance_test.cpp:106-128 (1000 batches, seed 1002)"""
    rng = O.Rng(1002)
    for _ in range(1000):
        n = 1 + rng() % 4
        s = 2 + rng() % 31
        d = 1 + rng() % 16
        st = rng.stack(n, s, d)
        rows = rng() % 32
        xs = rng.matrix(rows, d)
        payload, _ = st.quantize_batch(xs)
        codes = st.unpack(payload, rows)
        for r in range(rows):
            assert list(codes[r]) == list(st.quantize(xs[r])[0])


def test_acceptance_4_blockwise():
    """acceptance_test.cpp:132-180 (seed 1003)"""
    rng = O.Rng(1003)
    for _ in range(50):
        n = 1 + rng() % 4
        st = rng.stack(n, 8, 6)
        rows = 1 + rng() % 40
        payload, _ = st.quantize_batch(rng.matrix(rows, 6))
        full = st.reconstruct_block(payload, rows, 0, rows)
        b = 0
        while b < rows:
            e = min(rows, b + 1 + rng() % 7)
            assert np.array_equal(st.reconstruct_block(payload, rows, b, e), full[b:e])
            b = e
    worst = 0.0
    for _ in range(100):
        ks = rng.stack(1 + rng() % 3, 8, 8, O.KEY)
        vs = rng.stack(1 + rng() % 3, 8, 8, O.VALUE)
        init, local = rng() % 5, 1 + rng() % 8
        c = O.Cache(ks, vs, init, local)
        n = 1 + rng() % 60
        c.prefill(rng.matrix(n, 8), rng.matrix(n, 8))
        q = rng.matrix(1, 8)[0]
        whole = c.attend(q, c.counts()["total"])
        for br in (1, 7):
            worst = max(worst, float(np.abs(c.attend(q, br) - whole).max()))
    assert worst <= 1e-6


def test_acceptance_5_window_accounting():
    """acceptance_test.cpp:184-220 (seed 1004)"""
    rng = O.Rng(1004)
    ks = rng.stack(2, 16, 16, O.KEY)
    vs = rng.stack(2, 16, 16, O.VALUE)
    c = O.Cache(ks, vs, 4, 1024)
    c.prefill(rng.matrix(2048, 16), rng.matrix(2048, 16))
    cnt = c.counts()
    assert (cnt["total"], cnt["compressed"], cnt["init"], cnt["local"]) == (2048, 1020, 4, 1024)
    for t in range(5000):
        c.append_token(rng.matrix(1, 16)[0], rng.matrix(1, 16)[0])
        cnt = c.counts()
        assert cnt["total"] == 2048 + t + 1
        assert cnt["batched"] == (t + 1) // 1024
    assert c.counts()["batched"] == 4 and c.counts()["total"] == 7048


# ---------------- Eigen arithmetic restatement sanity ----------------

def test_effective_matches_row_major_product():
    """codebook.cpp:30-39: effective = entries . projection^T (fp32 GEMV order)."""
    st = O.Rng(77).stack(2, 32, 128)
    for s in range(2):
        ref = st.entries(s).astype(np.float64) @ st.projection(s).astype(np.float64).T
        np.testing.assert_allclose(st.effective(s), ref, rtol=1e-4, atol=1e-5)
        np.testing.assert_allclose(st.sqnorm(s), (st.effective(s).astype(np.float64) ** 2).sum(1), rtol=1e-5)


def test_generator_deterministic():
    """synthetic.cpp:40-63: same seed, same data; rope rotation preserves pair norms."""
    a = O.generate(O.ROPE_ROTATED_KEYS, 16, 5, 4, 9)
    b = O.generate(O.ROPE_ROTATED_KEYS, 16, 5, 4, 9)
    g = O.generate(O.GAUSSIAN_MIXTURE, 16, 5, 4, 9)
    assert np.array_equal(a, b)
    np.testing.assert_allclose(
        np.hypot(a[:, 0::2], a[:, 1::2]), np.hypot(g[:, 0::2], g[:, 1::2]), rtol=1e-5
    )
