"""Device-resident, batched CacheState.

Mirrors the reference's three-segment KV store (proj/core/include/vqkv/kv_cache.hpp:45-108,
proj/core/src/kv_cache.cpp:41-204) for `n_streams` (sequence, layer, KV head) streams that
advance in lockstep, the way a decoding model steps all of its streams together:

    init (raw prompt head, <= init_len rows) | compressed middle (CodeMatrix payload)
    | pending (raw, evicted from the window, not yet encoded) | local (raw window, local_len)

Everything lives in HBM.  Compressed rows are encoded by the tensor-core encoder
(`quantize_streams`, kv_cache.cpp:87-88 / :109-110) and appended to fixed-capacity payload
buffers with `vqkv_payload_append`; pending + local rows share one contiguous raw tail buffer
of 2 * local_len rows, so a flush is one batched encode of the first `pending` rows
(kv_cache.cpp:102-120) and attention reads every segment in place (strided views, no copies).

When the key stack has an attention layout (D = 128, <= 1024 entries per stage) the key codes
are kept ONLY as attention records (include/vqkv_c.h, vqkv_keycodes_to_gm: 10 B per token and
group of 8 key stages, the CodeMatrix row's 70 B at the paper geometry): each flush transcodes its
new rows once, decode attention reads them directly, and the CodeMatrix rows the reference API
exposes (codes, view_block, fidelity, snapshots) are rebuilt on demand by vqkv_keycodes_from_gm.
Value codes stay CodeMatrix rows (the attention kernel reads them as they are).

Semantics follow the reference exactly: prefill split (kv_cache.cpp:61-100), eviction to
pending and deferred (or eager) flush at local_len pending rows (:122-141), token order of
view_block (:143-189), memory accounting (:191-204), error kinds and messages.
"""
from __future__ import annotations

from typing import Dict, Optional, Tuple

import torch

from . import _lib
from . import device as Dv
from .errors import InvalidInput, InvalidState

__all__ = ["DeviceCacheState"]


class DeviceCacheState:
    """Batched CacheState on one GPU: n_streams streams with identical token counts."""

    def __init__(self, key_stack, value_stack, n_streams: int, init_len: int = 4, local_len: int = 1024,
                 eager: bool = False, device: Optional[torch.device] = None, capacity_rows: int = 0,
                 attn_layout: str = "auto"):
        if local_len < 1:  # WindowPolicy::validate (kv_cache.cpp:41-45)
            raise InvalidInput("local_len must be >= 1")
        if n_streams < 1:
            raise InvalidInput("n_streams must be >= 1")
        self.kstack, self.vstack = key_stack, value_stack
        self.kd, self.vd = Dv._dev(key_stack), Dv._dev(value_stack)
        self.n_streams = int(n_streams)
        self.init_len, self.local_len, self.eager = int(init_len), int(local_len), bool(eager)
        self.device = torch.device("cuda", self.kd.device) if device is None else torch.device(device)
        S, Dk, Dvv = self.n_streams, self.kd.dim, self.vd.dim
        f32 = dict(dtype=torch.float32, device=self.device)
        self.init_k = torch.zeros((S, max(self.init_len, 1), Dk), **f32)
        self.init_v = torch.zeros((S, max(self.init_len, 1), Dvv), **f32)
        self.tail_k = torch.zeros((S, 2 * self.local_len, Dk), **f32)
        self.tail_v = torch.zeros((S, 2 * self.local_len, Dvv), **f32)
        self.n_init = 0
        self.n_comp = 0
        self.n_tail = 0          # pending + local rows in the tail buffer
        self.prefilled = False
        self.batched = 0         # flush_pending count (kv_cache.hpp: batched_compressions_)
        self.cap_rows = 0
        self.kpay = self.vpay = None
        self.knorm = self.vnorm = None
        # attention layout of the key codes: "group_major" mirror, or "rows" (the payload itself)
        if attn_layout not in ("auto", "rows", "group_major"):
            raise InvalidInput("attn_layout must be 'auto', 'rows' or 'group_major'")
        gm_ok = Dv.keycodes_gm_bytes(self.kd, Dv.GM_ALIGN) > 0
        if attn_layout == "group_major" and not gm_ok:
            raise InvalidInput("the key stack has no group-major layout (D = 128, <= 1024 entries per stage)")
        self.attn_layout = "group_major" if (attn_layout != "rows" and gm_ok) else "rows"
        self.kgm, self.gm_cap = None, 0
        self._grow(max(int(capacity_rows), 0))

    # ---- geometry ---------------------------------------------------------
    @property
    def pending(self) -> int:
        return max(0, self.n_tail - self.local_len)

    @property
    def local(self) -> int:
        return self.n_tail - self.pending

    def total_len(self) -> int:
        return self.n_init + self.n_comp + self.n_tail

    def counts(self) -> Dict[str, int]:
        return dict(init=self.n_init, compressed=self.n_comp, pending=self.pending, local=self.local,
                    total=self.total_len(), batched=self.batched)

    def _grow(self, rows: int) -> None:
        """Make room for `rows` compressed rows per stream (capacity doubles)."""
        if rows <= self.cap_rows and self.vpay is not None:
            return
        cap = max(rows, 2 * self.cap_rows, 1024)
        vb = self.vd.payload_bytes(cap)
        # zero-filled: payload_append ORs into the first partial byte
        vpay = torch.zeros((self.n_streams, vb), dtype=torch.uint8, device=self.device)
        knorm = torch.zeros((self.n_streams, cap), dtype=torch.float32, device=self.device)
        vnorm = torch.zeros((self.n_streams, cap), dtype=torch.float32, device=self.device)
        if self.vpay is not None and self.n_comp:
            ovb = self.vd.payload_bytes(self.n_comp)
            vpay[:, :ovb] = self.vpay[:, :ovb]
            knorm[:, : self.n_comp] = self.knorm[:, : self.n_comp]
            vnorm[:, : self.n_comp] = self.vnorm[:, : self.n_comp]
        if self.attn_layout == "group_major":
            # the key codes live ONLY as attention records: per key group a u64 plane and a u16
            # plane of gm_cap tokens each; growing copies the first n_comp tokens of every plane
            gm_cap = -(-cap // Dv.GM_ALIGN) * Dv.GM_ALIGN
            ng = Dv.keycodes_gm_bytes(self.kd, Dv.GM_ALIGN) // (10 * Dv.GM_ALIGN)
            kgm = torch.zeros((self.n_streams, Dv.keycodes_gm_bytes(self.kd, gm_cap)), dtype=torch.uint8,
                              device=self.device)
            if self.kgm is not None and self.n_comp:
                n, oc = self.n_comp, self.gm_cap
                old = self.kgm.view(self.n_streams, ng, oc * 10)
                new = kgm.view(self.n_streams, ng, gm_cap * 10)
                new[:, :, : n * 8] = old[:, :, : n * 8]
                new[:, :, gm_cap * 8: gm_cap * 8 + n * 2] = old[:, :, oc * 8: oc * 8 + n * 2]
            self.kgm, self.gm_cap = kgm, gm_cap
        else:
            kb = self.kd.payload_bytes(cap)
            kpay = torch.zeros((self.n_streams, kb), dtype=torch.uint8, device=self.device)
            if self.kpay is not None and self.n_comp:
                ob = self.kd.payload_bytes(self.n_comp)
                kpay[:, :ob] = self.kpay[:, :ob]
            self.kpay = kpay
        self.vpay, self.knorm, self.vnorm, self.cap_rows = vpay, knorm, vnorm, cap

    def _encode_append(self, keys: torch.Tensor, values: torch.Tensor) -> None:
        """quantize_batch of [S, n, D] rows and CodeMatrix::append of the result."""
        n = keys.shape[1]
        if n == 0:
            return
        self._grow(self.n_comp + n)
        kp, kn = Dv.quantize_streams(self.kstack, keys.contiguous())
        vp, vn = Dv.quantize_streams(self.vstack, values.contiguous())
        stream = Dv._stream(keys)
        appends = [(self.vpay, vp, self.vd.row_bits)]
        if self.kgm is not None:  # key rows -> attention records at token n_comp
            Dv.keycodes_to_gm(self.kstack, kp, n, gm=self.kgm, cap=self.gm_cap, dst_row=self.n_comp)
        else:
            appends.append((self.kpay, kp, self.kd.row_bits))
        for pay, src, rb in appends:
            _lib.call("vqkv_payload_append", pay.data_ptr(), pay.stride(0), self.n_comp * rb, src.data_ptr(),
                      src.stride(0), n * rb, self.n_streams, stream)
        self.knorm[:, self.n_comp: self.n_comp + n] = kn
        self.vnorm[:, self.n_comp: self.n_comp + n] = vn
        self.n_comp += n

    def _check_rows(self, keys: torch.Tensor, values: torch.Tensor, ndim: int) -> None:
        for t, nm in ((keys, "keys"), (values, "values")):
            if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or t.device != self.device:
                raise InvalidInput(f"{nm} must be float32 tensors on {self.device}")
            if t.dim() != ndim or t.shape[0] != self.n_streams:
                raise InvalidInput(f"{nm} must have shape [n_streams, ...] with n_streams = {self.n_streams}")

    # ---- writers (single writer, kv_cache.hpp:41-44) ----------------------
    def prefill(self, keys: torch.Tensor, values: torch.Tensor) -> None:
        """keys [S, L, Dk], values [S, L, Dv] -> init | compressed | local (kv_cache.cpp:61-100)."""
        if self.total_len() != 0 or self.prefilled:
            raise InvalidState("prefill requires an empty cache")
        self._check_rows(keys, values, 3)
        if keys.shape[1] < 1:
            raise InvalidInput("prefill needs at least one token")
        if keys.shape[1] != values.shape[1]:
            raise InvalidInput("keys and values must have the same length")
        if keys.shape[2] != self.kd.dim or values.shape[2] != self.vd.dim:
            raise InvalidInput("key/value dimensions do not match the stacks")
        L = keys.shape[1]
        n_init = min(self.init_len, L)
        n_local = min(self.local_len, L - n_init)
        n_mid = L - n_init - n_local
        self.init_k[:, :n_init] = keys[:, :n_init]
        self.init_v[:, :n_init] = values[:, :n_init]
        self.n_init = n_init
        if n_mid > 0:
            self._encode_append(keys[:, n_init:n_init + n_mid], values[:, n_init:n_init + n_mid])
        self.tail_k[:, :n_local] = keys[:, L - n_local:]
        self.tail_v[:, :n_local] = values[:, L - n_local:]
        self.n_tail = n_local
        self.prefilled = True

    def append_token(self, keys: torch.Tensor, values: torch.Tensor) -> None:
        """keys [S, Dk], values [S, Dv]: one decode step for every stream (kv_cache.cpp:122-141)."""
        if not self.prefilled and self.init_len != 0:
            raise InvalidState("append_token requires a prefilled cache (or init_len == 0)")
        self._check_rows(keys, values, 2)
        if keys.shape[1] != self.kd.dim or values.shape[1] != self.vd.dim:
            raise InvalidInput("key/value dimensions do not match the stacks")
        self.tail_k[:, self.n_tail] = keys
        self.tail_v[:, self.n_tail] = values
        self.n_tail += 1
        if self.n_tail > self.local_len and (self.eager or self.pending >= self.local_len):
            self.flush_pending()

    def flush_pending(self) -> None:
        """Encode the pending rows as one batch and append them (kv_cache.cpp:102-120)."""
        p = self.pending
        if p == 0:
            return
        self._encode_append(self.tail_k[:, :p], self.tail_v[:, :p])
        rest = self.n_tail - p
        self.tail_k[:, :rest] = self.tail_k[:, p:self.n_tail].clone()
        self.tail_v[:, :rest] = self.tail_v[:, p:self.n_tail].clone()
        self.n_tail = rest
        self.batched += 1

    # ---- readers ------------------------------------------------------------
    def view_block(self, begin: int, end: int) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
        """Token rows [begin, end) of every stream -> (keys [S, n, Dk], values [S, n, Dv], exact [n])."""
        L = self.total_len()
        if begin < 0 or begin > end or end > L:
            raise InvalidInput(f"view range [{begin}, {end}) out of bounds for length {L}")
        S, n = self.n_streams, end - begin
        keys = torch.empty((S, n, self.kd.dim), dtype=torch.float32, device=self.device)
        values = torch.empty((S, n, self.vd.dim), dtype=torch.float32, device=self.device)
        exact = torch.ones(n, dtype=torch.bool)
        ie, ce = self.n_init, self.n_init + self.n_comp
        if begin < ie:
            e = min(end, ie)
            keys[:, : e - begin] = self.init_k[:, begin:e]
            values[:, : e - begin] = self.init_v[:, begin:e]
        if begin < ce and end > ie:
            b, e = max(begin, ie), min(end, ce)
            keys[:, b - begin: e - begin] = Dv.reconstruct_streams(self.kstack, self._payload(0), self.n_comp,
                                                                   b - ie, e - ie)
            values[:, b - begin: e - begin] = Dv.reconstruct_streams(self.vstack, self._payload(1), self.n_comp,
                                                                     b - ie, e - ie)
            exact[b - begin: e - begin] = False
            # an out-of-range code (a foreign payload) only sets the stack's sticky device flag:
            # surface it as the reference's InvalidCode (codebook.cpp:212-217)
            for st in (self.kd, self.vd):
                _lib.call("vqkv_stack_take_error", st.h)
        if end > ce:
            b = max(begin, ce)
            keys[:, b - begin:] = self.tail_k[:, b - ce: end - ce]
            values[:, b - begin:] = self.tail_v[:, b - ce: end - ce]
        return keys, values, exact

    def _payload(self, which: int) -> torch.Tensor:
        """CodeMatrix payload [S, payload_bytes(compressed)] of keys (0) / values (1); the key
        payload is rebuilt from the attention records when the cache keeps only those."""
        if which == 0 and self.kgm is not None:
            return Dv.keycodes_from_gm(self.kstack, self.kgm, self.gm_cap, self.n_comp)
        st, pay = (self.kd, self.kpay) if which == 0 else (self.vd, self.vpay)
        return pay[:, : max(st.payload_bytes(self.n_comp), 1)]

    def codes(self, which: int) -> Tuple[torch.Tensor, torch.Tensor]:
        """(payload [S, payload_bytes(compressed)] u8, residual norms [S, compressed]) of keys (0) / values (1)."""
        st = self.kd if which == 0 else self.vd
        pay = self._payload(which)[:, : st.payload_bytes(self.n_comp)]
        nrm = (self.knorm if which == 0 else self.vnorm)[:, : self.n_comp]
        return pay, nrm

    def memory_report(self) -> Dict[str, float]:
        """Per-stream accounting, kv_cache.cpp:191-204 (raw scalars counted at 2 bytes)."""
        spt = self.kd.dim + self.vd.dim
        bits = self.n_comp * (self.kd.row_bits + self.vd.row_bits)
        ratio = 1.0 - bits / float(self.n_comp * spt * 16) if self.n_comp else 0.0
        return dict(raw_bytes_equivalent=self.total_len() * spt * 2, compressed_payload_bits=bits,
                    codebook_overhead_bytes=self.kd.serialized_bytes() + self.vd.serialized_bytes(),
                    effective_ratio=ratio,
                    # device bytes per stream holding the compressed codes: key attention records
                    # (10 B per token and group of 8 key stages) or CodeMatrix rows, + value rows
                    device_code_bytes=(self.n_comp * 10 * (-(-self.kd.n // 8)) if self.kgm is not None
                                       else self.kd.payload_bytes(self.n_comp)) + self.vd.payload_bytes(self.n_comp))

    def attend(self, q: torch.Tensor, scale: float = 0.0, want_lse: bool = True):
        """Decode-step attention for q [S, G, Dk] over every segment, read in place
        (attention.cpp:26-69 over view_block order) -> (out [S, G, Dv], lse [S, G])."""
        if self.total_len() == 0:
            raise InvalidState("cannot attend over an empty cache")
        ni, nt = self.n_init, self.n_tail
        gm = (self.kgm is not None and self.n_comp > 0 and q.dim() == 3
              and Dv.attend_gm_supported(self.kstack, self.vstack, self.n_streams, q.shape[1], ni, self.n_comp, nt))
        return Dv.attend_decode(
            self.kstack, self.vstack, q,
            (self.kgm if gm else self._payload(0)) if self.n_comp else None, self.vpay if self.n_comp else None,
            self.n_comp,
            self.init_k[:, :ni] if ni else None, self.init_v[:, :ni] if ni else None,
            self.tail_k[:, :nt] if nt else None, self.tail_v[:, :nt] if nt else None,
            scale=scale, want_lse=want_lse, kcodes_gm_cap=self.gm_cap if gm else 0)

    def fidelity(self, original_keys: torch.Tensor, original_values: torch.Tensor, queries: torch.Tensor,
                 scale: float = 0.0) -> Dict[str, torch.Tensor]:
        """FidelityReport per stream (attention.cpp:90-134): attention over the cache against
        attention over the original rows, and the compressed rows' reconstruction MSE.

        original_keys [S, L, Dk] / original_values [S, L, Dv] (L = total_len), queries [S, Q, Dk].
        Returns float64 tensors [S]: output_max_abs_err, output_mean_cosine,
        key_intermediate_mse, value_intermediate_mse."""
        L = self.total_len()
        for t, nm, d in ((original_keys, "original_keys", self.kd.dim), (original_values, "original_values",
                                                                          self.vd.dim)):
            if t.dim() != 3 or t.shape[0] != self.n_streams or t.shape[1] != L:
                raise InvalidInput("originals length does not match cache length")
            if t.shape[2] != d:
                raise InvalidInput("originals dimensions do not match the cache")
        if queries.dim() != 3 or queries.shape[0] != self.n_streams or queries.shape[1] < 1 \
                or queries.shape[2] != self.kd.dim:
            raise InvalidInput("queries must be nonempty with the key dimension")
        # the reference runs one query at a time (attention.cpp:104-106); the kernels take the
        # queries as GQA groups, so they go in groups of 4 (the LUT kernel's G; the last group
        # is padded with copies of its first query, whose outputs are dropped)
        Q = queries.shape[1]
        comp_parts, raw_parts = [], []
        ok, ov = original_keys.contiguous(), original_values.contiguous()
        for q0 in range(0, Q, 4):
            qg = queries[:, q0:q0 + 4]
            n = qg.shape[1]
            if n < 4:
                qg = torch.cat([qg, qg[:, :1].expand(-1, 4 - n, -1)], dim=1)
            qg = qg.contiguous()
            c, _ = self.attend(qg, scale=scale, want_lse=False)
            # the reference's attend_raw over the originals: the same kernels with every row raw
            r, _ = Dv.attend_decode(self.kstack, self.vstack, qg, None, None, 0, None, None, ok, ov, scale=scale,
                                    want_lse=False)
            comp_parts.append(c[:, :n])
            raw_parts.append(r[:, :n])
        comp, raw = torch.cat(comp_parts, dim=1), torch.cat(raw_parts, dim=1)
        c64, r64 = comp.double(), raw.double()
        max_err = (comp - raw).abs().amax(dim=(1, 2)).double()
        cn, rn = c64.norm(dim=2), r64.norm(dim=2)
        denom = cn * rn
        cos = torch.where(denom > 0, (c64 * r64).sum(dim=2) / torch.where(denom > 0, denom, torch.ones_like(denom)),
                          ((cn == 0) & (rn == 0)).double())
        out = dict(output_max_abs_err=max_err, output_mean_cosine=cos.mean(dim=1),
                   key_intermediate_mse=torch.zeros(self.n_streams, dtype=torch.float64, device=self.device),
                   value_intermediate_mse=torch.zeros(self.n_streams, dtype=torch.float64, device=self.device))
        if self.n_comp > 0:
            f, n = self.n_init, self.n_comp
            rk = Dv.reconstruct_streams(self.kstack, self._payload(0), n, 0, n)
            rv = Dv.reconstruct_streams(self.vstack, self._payload(1), n, 0, n)
            dk = (original_keys[:, f:f + n] - rk).double()
            dvv = (original_values[:, f:f + n] - rv).double()
            out["key_intermediate_mse"] = (dk * dk).sum(dim=2).mean(dim=1)
            out["value_intermediate_mse"] = (dvv * dvv).sum(dim=2).mean(dim=1)
        return out

    # ---- VQKS snapshots (kv_cache.cpp:206-312), one file per stream ------------------
    def save_snapshot(self, stream: int, out) -> None:
        """Write stream `stream` as the reference's VQKS snapshot (byte layout of
        CacheState::save_snapshot).  `out` is a path or a binary file object."""
        import struct

        from .codebook import CodeMatrix, stack_content_hash
        from .errors import IoError

        if isinstance(out, str):
            try:
                with open(out, "wb") as f:
                    return self.save_snapshot(stream, f)
            except OSError as e:
                raise IoError(f"cannot open {out} for writing") from e
        if not 0 <= stream < self.n_streams:
            raise InvalidInput(f"stream {stream} out of range")
        i = stream
        w = out.write
        w(b"VQKS")
        w(struct.pack("<IQQBBQII", 1, self.init_len, self.local_len, int(self.eager), int(self.prefilled),
                      self.total_len(), self.kd.dim, self.vd.dim))
        w(struct.pack("<QQQ", stack_content_hash(self.kstack), stack_content_hash(self.vstack), self.batched))
        for t in (self.init_k, self.init_v):
            w(struct.pack("<Q", self.n_init))
            w(t[i, : self.n_init].contiguous().cpu().numpy().tobytes())
        for which, sizes in ((0, self.kd.sizes), (1, self.vd.sizes)):
            pay, _ = self.codes(which)
            CodeMatrix.from_payload(sizes, pay[i].cpu().numpy(), self.n_comp).save(out)
        w(self.knorm[i, : self.n_comp].contiguous().cpu().numpy().tobytes())
        w(self.vnorm[i, : self.n_comp].contiguous().cpu().numpy().tobytes())
        p = self.pending
        for t, a, b in ((self.tail_k, 0, p), (self.tail_v, 0, p), (self.tail_k, p, self.n_tail),
                        (self.tail_v, p, self.n_tail)):
            w(struct.pack("<Q", b - a))
            w(t[i, a:b].contiguous().cpu().numpy().tobytes())

    @classmethod
    def load_snapshots(cls, sources, key_stack, value_stack, device=None) -> "DeviceCacheState":
        """CacheState::load_snapshot of one VQKS file per stream into one batched cache.
        All snapshots must share policy and segment lengths (streams step in lockstep)."""
        import io
        import struct

        import numpy as np

        from .codebook import CodeMatrix, stack_content_hash
        from .errors import FormatError, InvalidCode, IoError

        parsed = []
        for src in sources:
            if isinstance(src, str):
                try:
                    with open(src, "rb") as f:
                        data = f.read()
                except OSError as e:
                    raise IoError(f"cannot open {src}") from e
            else:
                data = src.read()
            inp = io.BytesIO(data)
            off = 0

            def rd(fmt, what):
                nonlocal off
                n = struct.calcsize(fmt)
                b = inp.read(n)
                if len(b) != n:
                    raise FormatError(f"truncated file reading {what}", off)
                off += n
                return struct.unpack(fmt, b)[0]

            def rd_f32(count, dim, what):
                nonlocal off
                nb = 4 * count * dim
                b = inp.read(nb)
                if len(b) != nb:
                    raise FormatError(f"truncated file reading {what}", off)
                off += nb
                return np.frombuffer(b, np.float32).reshape(count, dim).copy()

            if inp.read(4) != b"VQKS":
                raise FormatError("bad magic (expected VQKS)", 0)
            off = 4
            version = rd("<I", "version")
            if version != 1:
                raise FormatError(f"unsupported snapshot version {version}", off - 4)
            init_len, local_len = rd("<Q", "init_len"), rd("<Q", "local_len")
            eager, prefilled = rd("<B", "eager flag") != 0, rd("<B", "prefilled flag") != 0
            stored_len = rd("<Q", "total_len")
            dk, dv = rd("<I", "key dim"), rd("<I", "value dim")
            if dk != key_stack.dim() or dv != value_stack.dim():
                raise InvalidInput("snapshot dimensions do not match the supplied stacks")
            kh, vh = rd("<Q", "key stack hash"), rd("<Q", "value stack hash")
            if kh != stack_content_hash(key_stack) or vh != stack_content_hash(value_stack):
                raise InvalidInput("snapshot was built against different codebook stacks")
            batched = rd("<Q", "compression count")
            init_k = rd_f32(rd("<Q", "init keys"), dk, "init keys")
            init_v = rd_f32(rd("<Q", "init values"), dv, "init values")
            kc, off = CodeMatrix.load(inp, off)
            vc, off = CodeMatrix.load(inp, off)
            # the codes must belong to the supplied stacks: same stage sizes and every index in
            # range (the reference rejects bad indices with InvalidCode when it decodes them,
            # codebook.cpp:212-217; the device decode would only raise a sticky flag)
            for cm, st in ((kc, key_stack), (vc, value_stack)):
                if list(cm.stage_sizes()) != [int(x) for x in st.stage_sizes()]:
                    raise InvalidInput("snapshot code stage sizes do not match the supplied stacks")
                if cm.rows():
                    codes = cm.all_rows()
                    bad = codes >= np.asarray(cm.stage_sizes(), dtype=codes.dtype)[None, :]
                    if bad.any():
                        r, st_i = map(int, np.argwhere(bad)[0])
                        raise InvalidCode(f"index {int(codes[r, st_i])} out of range for stage {st_i}")
            kn = rd_f32(kc.rows(), 1, "key residual norms")[:, 0]
            vn = rd_f32(vc.rows(), 1, "value residual norms")[:, 0]
            pend_k = rd_f32(rd("<Q", "pending keys"), dk, "pending keys")
            pend_v = rd_f32(rd("<Q", "pending values"), dv, "pending values")
            loc_k = rd_f32(rd("<Q", "local keys"), dk, "local keys")
            loc_v = rd_f32(rd("<Q", "local values"), dv, "local values")
            if len(init_k) + kc.rows() + len(pend_k) + len(loc_k) != stored_len:
                raise FormatError("segment lengths do not add up to total_len", off)
            parsed.append(dict(policy=(init_len, local_len, eager), prefilled=prefilled, batched=batched,
                               init=(init_k, init_v), codes=(kc, vc), norms=(kn, vn), pending=(pend_k, pend_v),
                               local=(loc_k, loc_v)))
        if not parsed:
            raise InvalidInput("no snapshots given")
        first = parsed[0]
        shape = lambda d: (d["policy"], d["prefilled"], d["batched"], len(d["init"][0]), d["codes"][0].rows(),
                           len(d["pending"][0]), len(d["local"][0]))
        if any(shape(d) != shape(first) for d in parsed):
            raise InvalidInput("snapshots of one batched cache must share policy and segment lengths")
        il, ll, eg = first["policy"]
        cache = cls(key_stack, value_stack, len(parsed), il, ll, eg, device, capacity_rows=first["codes"][0].rows())
        dev = cache.device
        t = lambda arrs: torch.from_numpy(np.stack(arrs)).to(dev)
        ni, nc = len(first["init"][0]), first["codes"][0].rows()
        npd, nl = len(first["pending"][0]), len(first["local"][0])
        if npd + nl > 2 * ll:
            raise FormatError("pending + local rows exceed the window capacity", 0)
        if ni:
            cache.init_k[:, :ni] = t([d["init"][0] for d in parsed])
            cache.init_v[:, :ni] = t([d["init"][1] for d in parsed])
        if nc:
            vb = cache.vd.payload_bytes(nc)
            kp = t([d["codes"][0].payload() for d in parsed])
            if cache.kgm is not None:
                Dv.keycodes_to_gm(key_stack, kp, nc, gm=cache.kgm, cap=cache.gm_cap)
            else:
                cache.kpay[:, : kp.shape[1]] = kp
            cache.vpay[:, :vb] = t([d["codes"][1].payload() for d in parsed])
            cache.knorm[:, :nc] = t([d["norms"][0] for d in parsed])
            cache.vnorm[:, :nc] = t([d["norms"][1] for d in parsed])
        for j, (a, b) in enumerate(((0, npd), (npd, npd + nl))):
            src = "pending" if j == 0 else "local"
            if b > a:
                cache.tail_k[:, a:b] = t([d[src][0] for d in parsed])
                cache.tail_v[:, a:b] = t([d[src][1] for d in parsed])
        cache.n_init, cache.n_comp, cache.n_tail = ni, nc, npd + nl
        cache.prefilled, cache.batched = first["prefilled"], first["batched"]
        return cache
