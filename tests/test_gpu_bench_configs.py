"""Parity at the benchmarked configurations (BASELINE.json configs[1] and configs[2]).

* configs[1]: 16,384 rope-rotated keys from the bench generator (synthetic.cpp:40-63, seed 1000
  + sid), through the paper's key stack (random_stack seed 1, 56 x 1024), on the tensor-core
  encoder.  Codes bit-exact except counted near-ties (tau of SURVEY.md 8c), residual norms
  bit-exact; the near-tie count is asserted to be reported and the mismatch count to be 0.
* configs[2]: full-size decode-step attention -- 2 (sequence, KV head) pairs x 131,072 tokens
  (4 init + 130,044 compressed + 1,024 local) x 4 query heads -- against the oracle's attend
  (attention.cpp:26-69, double precision) over the same segments, through both key-code
  layouts the library accepts.  Bar: max|o - o_ref| <= 2^-7 max(1, max|o_ref|).
"""
import os

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


def product_stack(o):
    from paper_2603_16435_b200 import codebook as P

    return P.CodebookStack.from_arrays([o.entries(s) for s in range(o.n)], [o.projection(s) for s in range(o.n)],
                                       o.kind)


def test_configs1_rope_keys_16k_bit_exact(torch_mod):
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    rows, init = 16384, 4
    ok = O.Rng(1).stack(56, 1024, 128, O.KEY)  # bench.make_stacks: vqkv_random_stack(seed 1)
    pk = product_stack(ok)
    # two bench streams (sid 0 and 1), rows after the 4 init rows, as bench.gen_inputs slices them
    xs = np.concatenate([O.generate(O.ROPE_ROTATED_KEYS, 128, rows // 2 + init, 32, 1000 + sid)[init:]
                         for sid in range(2)])
    x = torch.from_numpy(np.ascontiguousarray(xs.reshape(2, rows // 2, 128))).cuda()
    pay, nrm = Dv.quantize_streams(pk, x)
    torch.cuda.synchronize()
    codes, norms, ins = ok.quantize_rows_instrumented_mt(xs)
    got = np.concatenate([ok.unpack(pay[i].cpu().numpy(), rows // 2) for i in range(2)])
    res = O.classify_codes(got, codes, ins, ok.stage_max_norm())
    print(f"configs[1] rope keys: rows={res['rows_checked']} mismatches={res['mismatches']} "
          f"near_ties={res['near_ties']}")
    assert res["rows_checked"] == rows
    assert res["mismatches"] == 0, res
    same = (got == codes).all(axis=1)
    gn = nrm.cpu().numpy().reshape(-1)
    assert np.array_equal(gn[same].view(np.uint32), norms[same].view(np.uint32))


@pytest.mark.parametrize("layout", ["rows", "group_major"])
def test_configs2_full_context_attention(torch_mod, layout):
    torch = torch_mod
    from paper_2603_16435_b200 import device as Dv

    ctx, n_init, n_local, n_pairs, G = 131072, 4, 1024, 2, 4
    n_comp = ctx - n_init - n_local
    ok, ov = O.Rng(1).stack(56, 1024, 128, O.KEY), O.Rng(2).stack(16, 512, 128, O.VALUE)
    pk, pv = product_stack(ok), product_stack(ov)
    g = np.random.default_rng(2027)
    kc = np.stack([ok.pack(g.integers(0, 1024, (n_comp, 56)).astype(np.uint32)) for _ in range(n_pairs)])
    vc = np.stack([ov.pack(g.integers(0, 512, (n_comp, 16)).astype(np.uint32)) for _ in range(n_pairs)])
    f = lambda n: g.standard_normal((n_pairs, n, 128)).astype(np.float32)
    ik, iv, lk, lv = f(n_init), f(n_init), f(n_local), f(n_local)
    q = g.standard_normal((n_pairs, G, 128)).astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if layout == "rows":
        out, lse = Dv.attend_decode(pk, pv, t(q), t(kc), t(vc), n_comp, t(ik), t(iv), t(lk), t(lv))
    else:
        cap = -(-n_comp // Dv.GM_ALIGN) * Dv.GM_ALIGN
        gm = Dv.keycodes_to_gm(pk, t(kc), n_comp, cap=cap)
        out, lse = Dv.attend_decode(pk, pv, t(q), gm, t(vc), n_comp, t(ik), t(iv), t(lk), t(lv), kcodes_gm_cap=cap)
    out, lse = out.cpu().numpy(), lse.cpu().numpy()
    from concurrent.futures import ThreadPoolExecutor

    def one(pg):
        pi, gg = divmod(pg, G)
        ref, ref_lse = O.attend_segments(ok, ov, ik[pi], iv[pi], kc[pi], vc[pi], n_comp, lk[pi], lv[pi], q[pi, gg])
        dev = float(np.abs(out[pi, gg] - ref).max() / max(1.0, float(np.abs(ref).max())))
        return dev, abs(float(lse[pi, gg]) - ref_lse) / max(1.0, abs(ref_lse))

    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        res = list(ex.map(one, range(n_pairs * G)))
    worst = max(r[0] for r in res)
    print(f"configs[2] full context ({layout}): max dev {worst:.3e} (tol {ATT_TOL:.3e}), "
          f"max lse rel err {max(r[1] for r in res):.3e}")
    assert worst <= ATT_TOL
    assert max(r[1] for r in res) <= 1e-3
