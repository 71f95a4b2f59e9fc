"""ctypes wrapper around oracle/_build/liboracle.so -- TEST INFRASTRUCTURE ONLY.

The CPU oracle restates the reference (proj/core/src/*.cpp) in plain C++; see
oracle/vqkv_oracle.cpp for per-function citations.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module.  The product (paper_2603_16435_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")

KEY, VALUE = 0, 1
OK, INVALID_INPUT, INVALID_STATE, INVALID_CODE, FORMAT_ERROR, IO_ERROR = 0, 1, 2, 3, 4, 5


class OracleError(Exception):
    def __init__(self, code: int, msg: str, offset: int = 0):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.offset = offset


def build() -> str:
    """Compile the oracle with its Makefile (g++ only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "vqkv_oracle.cpp")
        ):
            build()
        L = C.CDLL(_SO)
        P = C.c_void_p
        fp = C.POINTER(C.c_float)
        u8p = C.POINTER(C.c_uint8)
        u32p = C.POINTER(C.c_uint32)
        u64p = C.POINTER(C.c_uint64)
        dp = C.POINTER(C.c_double)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_last_error_offset": (C.c_uint64, []),
            "orc_rng_new": (P, [C.c_uint64]),
            "orc_rng_free": (None, [P]),
            "orc_rng_next": (C.c_uint64, [P]),
            "orc_random_matrix": (None, [P, C.c_int64, C.c_int64, C.c_float, fp]),
            "orc_random_stack": (P, [P, C.c_uint32, C.c_uint32, C.c_int64, C.c_int]),
            "orc_stack_new": (P, [C.c_uint32, u32p, C.c_int64, fp, fp, C.c_int]),
            "orc_stack_free": (None, [P]),
            "orc_stack_num_stages": (C.c_uint32, [P]),
            "orc_stack_dim": (C.c_int64, [P]),
            "orc_stack_stage_size": (C.c_uint32, [P, C.c_uint32]),
            "orc_stack_kind": (C.c_int, [P]),
            "orc_stack_get_entries": (None, [P, C.c_uint32, fp]),
            "orc_stack_get_projection": (None, [P, C.c_uint32, fp]),
            "orc_stack_get_effective": (None, [P, C.c_uint32, fp]),
            "orc_stack_get_sqnorm": (None, [P, C.c_uint32, fp]),
            "orc_stack_save": (C.c_int, [P, C.c_char_p]),
            "orc_stack_serialize": (C.c_uint64, [P, u8p, C.c_uint64]),
            "orc_stack_load": (P, [C.c_char_p]),
            "orc_stack_load_bytes": (P, [u8p, C.c_uint64]),
            "orc_stack_hash": (C.c_uint64, [P]),
            "orc_index_bit_width": (C.c_uint, [C.c_uint32]),
            "orc_row_bits": (C.c_uint64, [C.c_uint32, u32p]),
            "orc_payload_bytes": (C.c_uint64, [C.c_uint32, u32p, C.c_uint64]),
            "orc_codes_pack": (C.c_int, [C.c_uint32, u32p, u32p, C.c_uint64, u8p]),
            "orc_codes_unpack": (C.c_int, [C.c_uint32, u32p, u8p, C.c_uint64, u32p]),
            "orc_nearest_entry": (C.c_int, [P, C.c_uint32, fp, C.c_int64, C.c_uint64, u32p, fp]),
            "orc_quantize": (C.c_int, [P, fp, C.c_int64, C.c_uint64, u32p, fp]),
            "orc_reconstruct": (C.c_int, [P, u32p, C.c_uint64, fp]),
            "orc_quantize_batch": (
                C.c_int,
                [P, fp, C.c_uint64, C.c_int64, C.c_uint64, u8p, fp, fp, fp, fp],
            ),
            "orc_quantize_batch_mt": (
                C.c_int,
                [P, fp, C.c_uint32, C.c_uint64, C.c_uint64, u8p, fp, C.c_int],
            ),
            "orc_reconstruct_block": (C.c_int, [P, u8p, C.c_uint64, C.c_uint64, C.c_uint64, fp]),
            "orc_stage_max_norm": (None, [P, fp]),
            "orc_generate": (
                C.c_int,
                [C.c_int, C.c_int64, C.c_int64, C.c_uint32, C.c_uint64, C.c_double, C.c_float, C.c_float, fp],
            ),
            "orc_cache_new": (P, [P, P, C.c_uint64, C.c_uint64, C.c_int]),
            "orc_cache_free": (None, [P]),
            "orc_cache_prefill": (C.c_int, [P, fp, fp, C.c_int64, C.c_int64, C.c_int64]),
            "orc_cache_append": (C.c_int, [P, fp, C.c_int64, fp, C.c_int64]),
            "orc_cache_counts": (None, [P, u64p]),
            "orc_cache_view_block": (C.c_int, [P, C.c_uint64, C.c_uint64, fp, fp, u8p]),
            "orc_cache_codes": (None, [P, C.c_int, u8p, fp]),
            "orc_cache_memory_report": (None, [P, u64p, u64p, u64p, dp]),
            "orc_attend": (C.c_int, [P, fp, C.c_int64, C.c_uint64, C.c_double, fp, u64p, u64p]),
            "orc_attend_raw": (
                C.c_int,
                [fp, fp, C.c_int64, C.c_int64, C.c_int64, fp, C.c_int64, C.c_double, fp],
            ),
            "orc_train_batch": (C.c_int, [P, fp, C.c_uint64, C.c_float, C.c_float, C.c_int, fp, dp]),
            "orc_train": (P, [fp, C.c_uint64, C.c_int64, C.c_uint32, u32p, C.c_void_p, C.c_int, dp, dp]),
            "orc_attend_segments": (
                C.c_int,
                [P, P, fp, fp, C.c_uint64, u8p, u8p, C.c_uint64, fp, fp, C.c_uint64, fp,
                 C.c_double, C.c_uint64, fp, dp],
            ),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _f(a):
    return a.ctypes.data_as(C.POINTER(C.c_float)) if a is not None else None


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8)) if a is not None else None


def _u32(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32)) if a is not None else None


def _check(status):
    if status != OK:
        L = lib()
        raise OracleError(status, L.orc_last_error().decode(), L.orc_last_error_offset())


def f32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a if shape is None else a.reshape(shape)


class Rng:
    """std::mt19937_64 (libstdc++), test_util.hpp fixtures."""

    def __init__(self, seed: int):
        self.h = lib().orc_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.orc_rng_free(self.h)
            except Exception:
                pass

    def __call__(self) -> int:
        return lib().orc_rng_next(self.h)

    def matrix(self, rows, cols, scale=1.0):
        out = np.empty((rows, cols), np.float32)
        lib().orc_random_matrix(self.h, rows, cols, scale, _f(out))
        return out

    def stack(self, n, size, dim, kind=KEY):
        return Stack(lib().orc_random_stack(self.h, n, size, dim, kind))


class Stack:
    def __init__(self, handle):
        if not handle:
            L = lib()
            raise OracleError(FORMAT_ERROR, L.orc_last_error().decode(), L.orc_last_error_offset())
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.orc_stack_free(self.h)
            except Exception:
                pass

    @classmethod
    def from_entries(cls, per_stage, projections=None, kind=KEY):
        """test_util.hpp:15-28 stack_from_entries (identity projections) or raw."""
        per_stage = [f32(e) for e in per_stage]
        dim = per_stage[0].shape[1]
        sizes = np.array([e.shape[0] for e in per_stage], np.uint32)
        ent = np.ascontiguousarray(np.concatenate([e.reshape(-1) for e in per_stage]))
        proj = None if projections is None else f32(np.stack(projections))
        return cls(lib().orc_stack_new(len(per_stage), _u32(sizes), dim, _f(ent), _f(proj), kind))

    @classmethod
    def load(cls, path):
        return cls(lib().orc_stack_load(path.encode()))

    @classmethod
    def from_bytes(cls, b: bytes):
        buf = np.frombuffer(b, np.uint8).copy()
        return cls(lib().orc_stack_load_bytes(_u8(buf), len(buf)))

    @property
    def n(self):
        return lib().orc_stack_num_stages(self.h)

    @property
    def dim(self):
        return lib().orc_stack_dim(self.h)

    @property
    def kind(self):
        return lib().orc_stack_kind(self.h)

    @property
    def sizes(self):
        return np.array([lib().orc_stack_stage_size(self.h, i) for i in range(self.n)], np.uint32)

    def _get(self, fn, stage, shape):
        out = np.empty(shape, np.float32)
        fn(self.h, stage, _f(out))
        return out

    def entries(self, s):
        return self._get(lib().orc_stack_get_entries, s, (int(self.sizes[s]), self.dim))

    def projection(self, s):
        return self._get(lib().orc_stack_get_projection, s, (self.dim, self.dim))

    def effective(self, s):
        return self._get(lib().orc_stack_get_effective, s, (int(self.sizes[s]), self.dim))

    def sqnorm(self, s):
        return self._get(lib().orc_stack_get_sqnorm, s, (int(self.sizes[s]),))

    def all_entries(self):
        return np.concatenate([self.entries(s).reshape(-1) for s in range(self.n)])

    def all_projections(self):
        return np.stack([self.projection(s) for s in range(self.n)])

    def stage_max_norm(self):
        out = np.empty(self.n, np.float32)
        lib().orc_stage_max_norm(self.h, _f(out))
        return out

    def save(self, path):
        _check(lib().orc_stack_save(self.h, path.encode()))

    def to_bytes(self) -> bytes:
        n = lib().orc_stack_serialize(self.h, None, 0)
        if n == 0:
            _check(INVALID_INPUT)
        buf = np.empty(n, np.uint8)
        lib().orc_stack_serialize(self.h, _u8(buf), n)
        return buf.tobytes()

    def hash(self) -> int:
        return lib().orc_stack_hash(self.h)

    # -- codebook.cpp:158-250 --
    def row_bits(self):
        s = self.sizes
        return lib().orc_row_bits(len(s), _u32(s))

    def payload_bytes(self, rows):
        s = self.sizes
        return lib().orc_payload_bytes(len(s), _u32(s), rows)

    def nearest_entry(self, stage, x, search_block=4096):
        x = f32(x)
        idx = C.c_uint32()
        dist = C.c_float()
        _check(lib().orc_nearest_entry(self.h, stage, _f(x), x.size, search_block, C.byref(idx), C.byref(dist)))
        return idx.value, dist.value

    def quantize(self, x, search_block=4096):
        x = f32(x)
        codes = np.empty(self.n, np.uint32)
        res = np.empty(max(self.dim, 1), np.float32)
        _check(lib().orc_quantize(self.h, _f(x), x.size, search_block, _u32(codes), _f(res)))
        return codes, res

    def reconstruct(self, codes):
        codes = np.ascontiguousarray(codes, np.uint32)
        out = np.empty(self.dim, np.float32)
        _check(lib().orc_reconstruct(self.h, _u32(codes), codes.size, _f(out)))
        return out

    def quantize_batch(self, xs, search_block=4096, instrument=False):
        xs = f32(xs)
        rows = xs.shape[0]
        xdim = xs.shape[1] if xs.ndim == 2 else 0
        payload = np.zeros(max(self.payload_bytes(rows), 1), np.uint8)
        norms = np.empty(max(rows, 1), np.float32)
        best = second = rn = None
        if instrument:
            best = np.empty((rows, self.n), np.float32)
            second = np.empty((rows, self.n), np.float32)
            rn = np.empty((rows, self.n), np.float32)
        _check(
            lib().orc_quantize_batch(
                self.h, _f(xs), rows, xdim, search_block, _u8(payload), _f(norms), _f(best), _f(second), _f(rn)
            )
        )
        payload = payload[: self.payload_bytes(rows)]
        if instrument:
            return payload, norms[:rows], dict(best=best, second=second, rnorm=rn)
        return payload, norms[:rows]

    def quantize_batch_mt(self, xs, n_streams, rows_per_stream, threads, search_block=4096):
        xs = f32(xs)
        pb = self.payload_bytes(rows_per_stream)
        payload = np.zeros(max(pb * n_streams, 1), np.uint8)
        norms = np.empty(max(n_streams * rows_per_stream, 1), np.float32)
        _check(
            lib().orc_quantize_batch_mt(
                self.h, _f(xs), n_streams, rows_per_stream, search_block, _u8(payload), _f(norms), threads
            )
        )
        return payload[: pb * n_streams], norms[: n_streams * rows_per_stream]

    def quantize_rows_instrumented_mt(self, xs, threads=None, chunk=256, search_block=4096):
        """quantize_batch of every row (codebook.cpp:225-237) with the per-stage instrumentation
        the near-tie rule needs, spread over host threads (ctypes releases the GIL; rows are
        independent, codebook.cpp:230-235).  Returns (codes [rows, n] u32, norms [rows],
        dict(best, second, rnorm) [rows, n])."""
        from concurrent.futures import ThreadPoolExecutor

        xs = f32(xs)
        rows = xs.shape[0]
        threads = threads or (os.cpu_count() or 1)
        codes = np.empty((rows, self.n), np.uint32)
        norms = np.empty(rows, np.float32)
        best = np.empty((rows, self.n), np.float32)
        second = np.empty((rows, self.n), np.float32)
        rn = np.empty((rows, self.n), np.float32)

        def one(r0):
            r1 = min(rows, r0 + chunk)
            pay, nrm, ins = self.quantize_batch(xs[r0:r1], search_block, instrument=True)
            codes[r0:r1] = self.unpack(pay, r1 - r0)
            norms[r0:r1] = nrm
            best[r0:r1], second[r0:r1], rn[r0:r1] = ins["best"], ins["second"], ins["rnorm"]

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, range(0, rows, chunk)))
        return codes, norms, dict(best=best, second=second, rnorm=rn)

    def reconstruct_block(self, payload, rows, begin, end):
        payload = np.ascontiguousarray(payload, np.uint8)
        if payload.size == 0:
            payload = np.zeros(1, np.uint8)
        out = np.empty((max(end - begin, 0), self.dim), np.float32)
        _check(lib().orc_reconstruct_block(self.h, _u8(payload), rows, begin, end, _f(out)))
        return out

    def pack(self, codes):
        s = self.sizes
        codes = np.ascontiguousarray(codes, np.uint32)
        rows = codes.shape[0]
        out = np.zeros(max(self.payload_bytes(rows), 1), np.uint8)
        _check(lib().orc_codes_pack(len(s), _u32(s), _u32(codes), rows, _u8(out)))
        return out[: self.payload_bytes(rows)]

    def unpack(self, payload, rows):
        s = self.sizes
        payload = np.ascontiguousarray(payload, np.uint8)
        if payload.size == 0:
            payload = np.zeros(1, np.uint8)
        out = np.empty((rows, len(s)), np.uint32)
        _check(lib().orc_codes_unpack(len(s), _u32(s), _u8(payload), rows, _u32(out)))
        return out


def index_bit_width(size):
    return lib().orc_index_bit_width(size)


def pack_codes(sizes, codes):
    sizes = np.ascontiguousarray(sizes, np.uint32)
    codes = np.ascontiguousarray(codes, np.uint32)
    rows = codes.shape[0]
    nb = lib().orc_payload_bytes(len(sizes), _u32(sizes), rows)
    out = np.zeros(max(nb, 1), np.uint8)
    _check(lib().orc_codes_pack(len(sizes), _u32(sizes), _u32(codes), rows, _u8(out)))
    return out[:nb]


def unpack_codes(sizes, payload, rows):
    sizes = np.ascontiguousarray(sizes, np.uint32)
    payload = np.ascontiguousarray(payload, np.uint8)
    if payload.size == 0:
        payload = np.zeros(1, np.uint8)
    out = np.empty((rows, len(sizes)), np.uint32)
    _check(lib().orc_codes_unpack(len(sizes), _u32(sizes), _u8(payload), rows, _u32(out)))
    return out


GAUSSIAN_MIXTURE, ROPE_ROTATED_KEYS = 0, 1


def generate(kind, dim, count, component_count=8, seed=0, rope_base=10000.0, component_std=0.25, mean_scale=1.0):
    out = np.empty((count, dim), np.float32)
    _check(lib().orc_generate(kind, dim, count, component_count, seed, rope_base, component_std, mean_scale, _f(out)))
    return out


class Cache:
    """kv_cache.hpp:45-108 CacheState restated."""

    def __init__(self, kstack: Stack, vstack: Stack, init_len=4, local_len=1024, eager=False):
        self.k, self.v = kstack, vstack  # keep alive
        h = lib().orc_cache_new(kstack.h, vstack.h, init_len, local_len, int(eager))
        if not h:
            _check(INVALID_INPUT)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.orc_cache_free(self.h)
            except Exception:
                pass

    def prefill(self, keys, values):
        keys, values = f32(keys), f32(values)
        _check(
            lib().orc_cache_prefill(
                self.h, _f(keys), _f(values), keys.shape[0], keys.shape[1] if keys.ndim == 2 else 0,
                values.shape[1] if values.ndim == 2 else 0,
            )
        )

    def append_token(self, key, value):
        key, value = f32(key), f32(value)
        _check(lib().orc_cache_append(self.h, _f(key), key.size, _f(value), value.size))

    def counts(self):
        o = np.zeros(6, np.uint64)
        lib().orc_cache_counts(self.h, o.ctypes.data_as(C.POINTER(C.c_uint64)))
        return dict(zip(["init", "compressed", "pending", "local", "total", "batched"], map(int, o)))

    def view_block(self, begin, end):
        n = max(end - begin, 0)
        k = np.empty((n, self.k.dim), np.float32)
        v = np.empty((n, self.v.dim), np.float32)
        ex = np.empty(max(n, 1), np.uint8)
        _check(lib().orc_cache_view_block(self.h, begin, end, _f(k), _f(v), _u8(ex)))
        return k, v, ex[:n].astype(bool)

    def codes(self, which):
        c = self.counts()["compressed"]
        st = self.k if which == 0 else self.v
        p = np.zeros(max(st.payload_bytes(c), 1), np.uint8)
        nrm = np.zeros(max(c, 1), np.float32)
        lib().orc_cache_codes(self.h, which, _u8(p), _f(nrm))
        return p[: st.payload_bytes(c)], nrm[:c]

    def memory_report(self):
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        r = C.c_double()
        lib().orc_cache_memory_report(self.h, C.byref(a), C.byref(b), C.byref(c), C.byref(r))
        return dict(raw_bytes_equivalent=a.value, compressed_payload_bits=b.value,
                    codebook_overhead_bytes=c.value, effective_ratio=r.value)

    def attend(self, q, block_rows=128, scale=0.0, stats=False):
        q = f32(q)
        out = np.empty(self.v.dim, np.float32)
        peak, nrec = C.c_uint64(0), C.c_uint64(0)
        _check(lib().orc_attend(self.h, _f(q), q.size, block_rows, scale, _f(out), C.byref(peak), C.byref(nrec)))
        if stats:
            return out, dict(peak_reconstructed_scalars=peak.value, reconstructed_rows=nrec.value)
        return out


def attend_raw(keys, values, q, scale=0.0):
    keys, values, q = f32(keys), f32(values), f32(q)
    out = np.empty(values.shape[1] if values.ndim == 2 else 1, np.float32)
    _check(
        lib().orc_attend_raw(
            _f(keys), _f(values), keys.shape[0], keys.shape[1] if keys.ndim == 2 else q.size,
            values.shape[1] if values.ndim == 2 else 1, _f(q), q.size, scale, _f(out),
        )
    )
    return out


def attend_segments(kst: Stack, vst: Stack, init_k, init_v, kpay, vpay, n_comp, local_k, local_v, q,
                    scale=0.0, block_rows=128):
    init_k, init_v, local_k, local_v, q = map(f32, (init_k, init_v, local_k, local_v, q))
    kpay = np.ascontiguousarray(kpay, np.uint8) if len(kpay) else np.zeros(1, np.uint8)
    vpay = np.ascontiguousarray(vpay, np.uint8) if len(vpay) else np.zeros(1, np.uint8)
    out = np.empty(vst.dim, np.float32)
    lse = C.c_double()
    _check(
        lib().orc_attend_segments(
            kst.h, vst.h, _f(init_k), _f(init_v), init_k.shape[0], _u8(kpay), _u8(vpay), n_comp,
            _f(local_k), _f(local_v), local_k.shape[0], _f(q), scale, block_rows, _f(out), C.byref(lse),
        )
    )
    return out, lse.value


def near_tie_tau(best, second, rnorm, emax):
    """tau = 2^-14 ||r|| max||e|| + 2^-22 max(|s1|, |s2|)."""
    return 2.0 ** -14 * rnorm * emax + 2.0 ** -22 * np.maximum(np.abs(best), np.abs(second))


def classify_codes(got, ref, ins, emax):
    """Per-row code parity against the oracle (north_star: bit-exact except reference near-ties).

    A row whose codes differ is a counted near-tie when, at its FIRST differing stage, the
    oracle's best/second-best score gap is <= tau (later stages of such a row follow a different
    residual and are excluded); otherwise it is a mismatch.
    Returns dict(rows_checked, mismatches, near_ties, mismatch_rows)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    bad = np.nonzero((got != ref).any(axis=1))[0]
    ties, mism = 0, []
    for r in bad:
        st = int(np.nonzero(got[r] != ref[r])[0][0])
        gap = float(ins["second"][r, st]) - float(ins["best"][r, st])
        tau = float(near_tie_tau(ins["best"][r, st], ins["second"][r, st], ins["rnorm"][r, st], emax[st]))
        if gap <= tau:
            ties += 1
        else:
            mism.append(int(r))
    return dict(rows_checked=int(got.shape[0]), mismatches=len(mism), near_ties=ties, mismatch_rows=mism[:16])


class TrainConfig(C.Structure):
    """orc_train_config (trainer.hpp TrainConfig, train_entries = false)."""

    _fields_ = [("learning_rate", C.c_float), ("batch_size", C.c_uint64), ("epochs", C.c_uint64), ("beta", C.c_float),
                ("gamma", C.c_float), ("seed", C.c_uint64), ("init_scale", C.c_float),
                ("square_commitment", C.c_int), ("holdout_fraction", C.c_float)]


def train_config(learning_rate=0.001, batch_size=65536, epochs=20, beta=0.25, gamma=1.0, seed=0, init_scale=1.0,
                 square_commitment=False, holdout_fraction=0.01):
    return TrainConfig(learning_rate, batch_size, epochs, beta, gamma, seed, init_scale, int(square_commitment),
                       holdout_fraction)


def train_batch(stack, batch, beta=0.25, gamma=1.0, square_commitment=False, grads=True):
    """accumulate_loss over one batch (trainer.cpp:36-86): (sums [3 + N], grad [N, D, D] or None)."""
    b = f32(batch)
    n, d = stack.n, stack.dim
    sums = np.zeros(3 + n, np.float64)
    g = np.zeros((n, d, d), np.float32) if grads else None
    _check(lib().orc_train_batch(stack.h, _f(b), b.shape[0], beta, gamma, int(square_commitment),
                                 _f(g) if grads else None, sums.ctypes.data_as(C.POINTER(C.c_double))))
    return sums, g


def train(data, stage_sizes, cfg, kind=KEY):
    """train() (trainer.cpp:166-248): (Stack, per_epoch_loss, per_stage_mse)."""
    x = f32(data)
    sizes = np.asarray(stage_sizes, np.uint32)
    el = np.zeros(int(cfg.epochs), np.float64)
    sm = np.zeros(len(sizes), np.float64)
    h = lib().orc_train(_f(x), x.shape[0], x.shape[1], len(sizes), sizes.ctypes.data_as(C.POINTER(C.c_uint32)),
                        C.byref(cfg), kind, el.ctypes.data_as(C.POINTER(C.c_double)),
                        sm.ctypes.data_as(C.POINTER(C.c_double)))
    if not h:
        raise OracleError(1, lib().orc_last_error().decode())
    return Stack(h), el, sm
