"""Python mirror of the reference codebook API (proj/core/include/vqkv/codebook.hpp).

Same names, argument meaning and error behaviour as the C++ reference; every
arithmetic operation runs in libvqkv_b200.so on the GPU (no CPU fallback).
Results are returned by value as numpy arrays, like the reference returns
Eigen matrices.  For batched, asynchronous, device-resident use see
:mod:`paper_2603_16435_b200.device`.
"""
from __future__ import annotations

import io
import struct
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .errors import FormatError, InvalidCode, InvalidInput, IoError

KEY, VALUE = 0, 1
DEFAULT_SEARCH_BLOCK = 4096  # codebook.hpp:25


def index_bit_width(size: int) -> int:
    """bitpack.hpp:38-45: ceil(log2 size), 0 for size 1."""
    w = 0
    while (1 << w) < size:
        w += 1
    return w


# --------------------------------------------------------------------------
# CodeMatrix (codebook.hpp:63-91, codebook.cpp:74-151)
# --------------------------------------------------------------------------
class CodeMatrix:
    """Append-only bit-packed rows; payload bytes identical to the reference."""

    def __init__(self, stage_sizes: Sequence[int] = ()):
        self._sizes = [int(s) for s in stage_sizes]
        for s in self._sizes:
            if s < 1:
                raise InvalidInput("stage size must be >= 1")
        self._bits = [index_bit_width(s) for s in self._sizes]
        self._offs = list(np.cumsum([0] + self._bits[:-1])) if self._bits else []
        self._row_bits = int(sum(self._bits))
        self._rows = 0
        self._payload = np.zeros(0, np.uint8)

    # -- accessors --
    def rows(self) -> int:
        return self._rows

    def num_stages(self) -> int:
        return len(self._sizes)

    def stage_sizes(self) -> List[int]:
        return list(self._sizes)

    def row_bits(self) -> int:
        return self._row_bits

    def payload_bits(self) -> int:
        return self._rows * self._row_bits

    def payload(self) -> np.ndarray:
        return self._payload

    def __eq__(self, other):
        return (
            isinstance(other, CodeMatrix)
            and self._sizes == other._sizes
            and self._rows == other._rows
            and np.array_equal(self._payload, other._payload)
        )

    # -- bulk helpers (vectorised) --
    @classmethod
    def from_payload(cls, stage_sizes, payload, rows):
        m = cls(stage_sizes)
        m._rows = int(rows)
        nb = (m._rows * m._row_bits + 7) // 8
        payload = np.ascontiguousarray(payload, np.uint8).reshape(-1)
        if payload.size < nb:
            raise InvalidInput("payload shorter than rows * row_bits")
        m._payload = payload[:nb].copy()
        return m

    def _codes_to_bits(self, codes: np.ndarray) -> np.ndarray:
        rows = codes.shape[0]
        bits = np.zeros((rows, self._row_bits), np.uint8)
        for s, (w, o) in enumerate(zip(self._bits, self._offs)):
            for b in range(w):
                bits[:, o + b] = (codes[:, s] >> b) & 1
        return bits.reshape(-1)

    def extend(self, codes) -> None:
        """append() for many rows at once (same validation)."""
        codes = np.asarray(codes, dtype=np.int64)
        if codes.ndim == 1:
            codes = codes.reshape(1, -1)
        if codes.shape[1] != len(self._sizes):
            raise InvalidInput("code vector has wrong stage count")
        for i, s in enumerate(self._sizes):
            bad = (codes[:, i] < 0) | (codes[:, i] >= s)
            if bad.any():
                raise InvalidCode(f"index {int(codes[bad, i][0])} out of range for stage {i}")
        codes = codes.astype(np.uint64)
        old_bits = self._rows * self._row_bits
        allbits = np.unpackbits(self._payload, bitorder="little")[:old_bits]
        allbits = np.concatenate([allbits, self._codes_to_bits(codes)])
        self._payload = np.packbits(allbits, bitorder="little")
        self._rows += codes.shape[0]

    def append(self, codes: Sequence[int]) -> None:
        self.extend(np.asarray(codes, dtype=np.int64).reshape(1, -1))

    def all_rows(self) -> np.ndarray:
        rows = self._rows
        bits = np.unpackbits(self._payload, bitorder="little", count=rows * self._row_bits)
        bits = bits.reshape(rows, self._row_bits).astype(np.uint32)
        out = np.zeros((rows, len(self._sizes)), np.uint32)
        for s, (w, o) in enumerate(zip(self._bits, self._offs)):
            for b in range(w):
                out[:, s] |= bits[:, o + b] << b
        return out

    def row(self, r: int) -> List[int]:
        if r < 0 or r >= self._rows:
            raise InvalidInput(f"row {r} out of range")
        bits = np.unpackbits(self._payload, bitorder="little", count=(r + 1) * self._row_bits)[
            r * self._row_bits :
        ]
        return [int(sum(int(bits[o + b]) << b for b in range(w))) for w, o in zip(self._bits, self._offs)]

    def code_at(self, r: int, stage: int) -> int:
        if r < 0 or r >= self._rows or stage < 0 or stage >= len(self._sizes):
            raise InvalidInput("code_at out of range")
        return self.row(r)[stage]

    # -- VQCM-style container body (codebook.cpp:125-151) --
    def save(self, out) -> None:
        out.write(struct.pack("<I", len(self._sizes)))
        for s in self._sizes:
            out.write(struct.pack("<I", s))
        out.write(struct.pack("<Q", self._rows))
        out.write(self._payload.tobytes())

    @classmethod
    def load(cls, inp, offset: int = 0):
        def rd(fmt, what):
            nonlocal offset
            n = struct.calcsize(fmt)
            b = inp.read(n)
            if len(b) != n:
                raise FormatError(f"truncated file reading {what}", offset)
            offset += n
            return struct.unpack(fmt, b)[0]

        n = rd("<I", "stage count")
        if n < 1:
            raise FormatError("stage count must be >= 1", offset - 4)
        sizes = []
        for _ in range(n):
            s = rd("<I", "stage size")
            if s < 1:
                raise FormatError("stage size must be >= 1", offset - 4)
            sizes.append(s)
        m = cls(sizes)
        m._rows = rd("<Q", "row count")
        nb = (m._rows * m._row_bits + 7) // 8
        b = inp.read(nb)
        if len(b) != nb:
            raise FormatError("truncated file reading code payload", offset)
        m._payload = np.frombuffer(b, np.uint8).copy()
        return m, offset + nb


# --------------------------------------------------------------------------
# Codebook / CodebookStack (codebook.hpp:30-56)
# --------------------------------------------------------------------------
@dataclass
class Codebook:
    entries: np.ndarray  # S x D
    projection: np.ndarray  # D x D
    effective: Optional[np.ndarray] = None  # S x D (device-computed)
    effective_sqnorm: Optional[np.ndarray] = None
    _single: object = field(default=None, repr=False, compare=False)

    def size(self) -> int:
        return int(self.entries.shape[0])

    def dim(self) -> int:
        return int(self.entries.shape[1])

    def validate(self) -> None:  # codebook.cpp:41-51
        if self.entries.ndim != 2 or self.size() < 1 or self.dim() < 1:
            raise InvalidInput("codebook must have S >= 1 and D >= 1")
        if self.projection.shape != (self.dim(), self.dim()):
            raise InvalidInput("projection must be DxD")
        if not (np.isfinite(self.entries).all() and np.isfinite(self.projection).all()):
            raise InvalidInput("codebook contains non-finite values")

    def refresh(self) -> None:
        """Recomputes effective entries + squared norms (on the GPU)."""
        self._single = None
        st = CodebookStack([self])
        self.effective, self.effective_sqnorm = st.device.effective(0)
        self._single = st


class CodebookStack:
    """Ordered residual stages; immutable once uploaded (codebook.hpp:45-56)."""

    def __init__(self, stages: Sequence[Codebook] = (), cache_kind: int = KEY, device: int = 0):
        self.stages = list(stages)
        self.cache_kind = cache_kind
        self._device_index = device
        self._dev = None

    def num_stages(self) -> int:
        return len(self.stages)

    def dim(self) -> int:
        return self.stages[0].dim() if self.stages else 0

    def stage_sizes(self) -> List[int]:
        return [c.size() for c in self.stages]

    def validate(self) -> None:  # codebook.cpp:62-72
        if not self.stages:
            raise InvalidInput("stack must have at least one stage")
        for c in self.stages:
            c.validate()
            if c.dim() != self.dim():
                raise InvalidInput("all stages must share one dimension")

    @property
    def device(self) -> "DeviceStack":
        if self._dev is None:
            self.validate()
            self._dev = DeviceStack(self, self._device_index)
            for i, c in enumerate(self.stages):
                if c.effective is None:
                    c.effective, c.effective_sqnorm = self._dev.effective(i)
        return self._dev

    def refresh(self) -> None:
        self._dev = None
        _ = self.device

    @classmethod
    def from_arrays(cls, entries: Sequence[np.ndarray], projections=None, cache_kind=KEY, device=0):
        projections = projections if projections is not None else [
            np.eye(np.asarray(e).shape[1], dtype=np.float32) for e in entries
        ]
        stages = [
            Codebook(np.ascontiguousarray(e, np.float32), np.ascontiguousarray(p, np.float32))
            for e, p in zip(entries, projections)
        ]
        st = cls(stages, cache_kind, device)
        _ = st.device
        return st


class DeviceStack:
    """Owns a vqkv_stack_t (device copy of one CodebookStack)."""

    def __init__(self, stack: CodebookStack, device: int = 0):
        import ctypes as C

        sizes = np.array(stack.stage_sizes(), np.uint32)
        ent = np.ascontiguousarray(np.concatenate([c.entries.reshape(-1) for c in stack.stages]), np.float32)
        proj = np.ascontiguousarray(np.stack([c.projection for c in stack.stages]), np.float32)
        h = C.c_void_p()
        _lib.call(
            "vqkv_stack_create",
            device,
            stack.cache_kind,
            len(sizes),
            sizes.ctypes.data_as(_lib.u32p),
            stack.dim(),
            ent.ctypes.data_as(_lib.fp),
            proj.ctypes.data_as(_lib.fp),
            C.byref(h),
        )
        self.h = h.value
        self.device = device
        self.n = len(sizes)
        self.dim = stack.dim()
        self.sizes = [int(s) for s in sizes]
        self.kind = stack.cache_kind
        self.row_bits = sum(index_bit_width(s) for s in self.sizes)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                _lib.load().vqkv_stack_destroy(h)
            except Exception:
                pass

    def payload_bytes(self, rows: int) -> int:
        return (rows * self.row_bits + 7) // 8

    def serialized_bytes(self) -> int:
        """RSVQ size of the stack (codebook.cpp:252-275): header + per stage S, D, entries, projection."""
        return 13 + sum(8 + 4 * (s * self.dim + self.dim * self.dim) for s in self.sizes)

    def effective(self, stage: int):
        e = np.empty((self.sizes[stage], self.dim), np.float32)
        q = np.empty(self.sizes[stage], np.float32)
        _lib.call("vqkv_stack_effective", self.h, stage, e.ctypes.data_as(_lib.fp), q.ctypes.data_as(_lib.fp))
        return e, q


# --------------------------------------------------------------------------
# Free functions (codebook.hpp:93-138)
# --------------------------------------------------------------------------
@dataclass
class NearestResult:
    index: int
    distance: float


@dataclass
class QuantizeResult:
    codes: List[int]
    final_residual: np.ndarray


@dataclass
class QuantizeBatchResult:
    codes: CodeMatrix
    residual_norms: np.ndarray


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_16435_b200 computes on a CUDA device; none is available")
    return torch


def _f32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def nearest_entry(codebook: Codebook, x, search_block: int = DEFAULT_SEARCH_BLOCK) -> NearestResult:
    """codebook.cpp:180-192"""
    x = _f32(x).reshape(-1)
    if x.size != codebook.dim():
        raise InvalidInput(f"vector dimension {x.size} does not match codebook dimension {codebook.dim()}")
    if not np.isfinite(x).all():
        raise InvalidInput("query vector contains non-finite values")
    if codebook._single is None:
        codebook.refresh()
    dev = codebook._single.device
    torch = _torch()
    xd = torch.from_numpy(x).to(f"cuda:{dev.device}")
    idx = torch.empty(1, dtype=torch.int32, device=xd.device)
    dist = torch.empty(1, dtype=torch.float32, device=xd.device)
    stream = torch.cuda.current_stream(xd.device).cuda_stream
    _lib.call("vqkv_nearest_batch", dev.h, 0, xd.data_ptr(), 1, search_block, idx.data_ptr(), dist.data_ptr(), stream)
    return NearestResult(int(idx.item()), float(dist.item()))


def _check_dim(stack: CodebookStack, got: int):
    if got != stack.dim():
        raise InvalidInput(f"vector dimension {got} does not match stack dimension {stack.dim()}")


def quantize_batch(stack: CodebookStack, xs, search_block: int = DEFAULT_SEARCH_BLOCK) -> QuantizeBatchResult:
    """codebook.cpp:225-237 -- row-for-row identical to quantize()."""
    xs = np.asarray(xs, dtype=np.float32)
    rows = xs.shape[0] if xs.ndim >= 1 else 0
    if rows > 0:
        _check_dim(stack, xs.shape[1] if xs.ndim == 2 else 1)
    cm = CodeMatrix(stack.stage_sizes())
    if rows == 0:
        return QuantizeBatchResult(cm, np.zeros(0, np.float32))
    payload, norms, _ = _quantize_rows(stack, xs, search_block, want_residuals=False)
    return QuantizeBatchResult(CodeMatrix.from_payload(stack.stage_sizes(), payload, rows), norms)


def _quantize_rows(stack: CodebookStack, xs: np.ndarray, search_block: int, want_residuals: bool):
    dev = stack.device
    torch = _torch()
    xd = torch.from_numpy(np.ascontiguousarray(xs, np.float32)).to(f"cuda:{dev.device}")
    rows = xs.shape[0]
    payload = torch.empty(max(dev.payload_bytes(rows), 1), dtype=torch.uint8, device=xd.device)
    norms = torch.empty(rows, dtype=torch.float32, device=xd.device)
    res = torch.empty((rows, dev.dim), dtype=torch.float32, device=xd.device) if want_residuals else None
    stream = torch.cuda.current_stream(xd.device).cuda_stream
    _lib.call(
        "vqkv_quantize_batch_ex", dev.h, xd.data_ptr(), 1, rows, search_block, payload.data_ptr(),
        norms.data_ptr(), res.data_ptr() if res is not None else None, stream,
    )
    return (
        payload.cpu().numpy()[: dev.payload_bytes(rows)],
        norms.cpu().numpy(),
        res.cpu().numpy() if res is not None else None,
    )


def quantize(stack: CodebookStack, x, search_block: int = DEFAULT_SEARCH_BLOCK) -> QuantizeResult:
    """codebook.cpp:194-206"""
    x = _f32(x).reshape(-1)
    _check_dim(stack, x.size)
    payload, _, res = _quantize_rows(stack, x.reshape(1, -1), search_block, want_residuals=True)
    codes = CodeMatrix.from_payload(stack.stage_sizes(), payload, 1).row(0)
    return QuantizeResult(codes, res[0])


def reconstruct_block(stack: CodebookStack, codes: CodeMatrix, begin: int, end: int) -> np.ndarray:
    """codebook.cpp:239-250 -- bit-exact stage-order sums."""
    if begin > end or end > codes.rows() or begin < 0:
        raise InvalidInput(f"row range [{begin}, {end}) out of bounds for {codes.rows()} rows")
    dev = stack.device
    if end == begin:
        return np.zeros((0, stack.dim()), np.float32)
    torch = _torch()
    pay = codes.payload()
    pd = torch.from_numpy(np.ascontiguousarray(pay) if pay.size else np.zeros(1, np.uint8)).to(f"cuda:{dev.device}")
    out = torch.empty((end - begin, dev.dim), dtype=torch.float32, device=pd.device)
    stream = torch.cuda.current_stream(pd.device).cuda_stream
    _lib.call("vqkv_reconstruct_block", dev.h, pd.data_ptr(), 1, codes.rows(), begin, end, out.data_ptr(), stream)
    st = _lib.load().vqkv_stack_take_error(dev.h)
    if st != 0:
        raise InvalidCode("code index out of range for its stage")
    return out.cpu().numpy()


def reconstruct(stack: CodebookStack, codes: Sequence[int]) -> np.ndarray:
    """codebook.cpp:208-223"""
    codes = [int(c) for c in codes]
    if len(codes) != stack.num_stages():
        raise InvalidCode(f"code vector has {len(codes)} stages, stack has {stack.num_stages()}")
    for i, (c, s) in enumerate(zip(codes, stack.stage_sizes())):
        if c < 0 or c >= s:
            raise InvalidCode(f"index {c} out of range for stage {i}")
    cm = CodeMatrix(stack.stage_sizes())
    cm.append(codes)
    return reconstruct_block(stack, cm, 0, 1)[0]


# --------------------------------------------------------------------------
# RSVQ container (codebook.cpp:252-336)
# --------------------------------------------------------------------------
def save_stack(stack: CodebookStack, out) -> None:
    if isinstance(out, str):
        try:
            with open(out, "wb") as f:
                save_stack(stack, f)
        except OSError as e:
            raise IoError(f"cannot open {out} for writing") from e
        return
    stack.validate()
    out.write(b"RSVQ")
    out.write(struct.pack("<IBI", 1, stack.cache_kind, stack.num_stages()))
    for c in stack.stages:
        out.write(struct.pack("<II", c.size(), c.dim()))
        out.write(np.ascontiguousarray(c.entries, np.float32).tobytes())
        out.write(np.ascontiguousarray(c.projection, np.float32).tobytes())


def load_stack(inp, device: int = 0) -> CodebookStack:
    if isinstance(inp, str):
        try:
            f = open(inp, "rb")
        except OSError as e:
            raise IoError(f"cannot open {inp}") from e
        with f:
            return load_stack(f, device)
    off = 0

    def rd(fmt, what):
        nonlocal off
        n = struct.calcsize(fmt)
        b = inp.read(n)
        if len(b) != n:
            raise FormatError(f"truncated file reading {what}", off)
        off += n
        return struct.unpack(fmt, b)[0]

    magic = inp.read(4)
    if magic != b"RSVQ":
        raise FormatError("bad magic, expected RSVQ", 0)
    off = 4
    version = rd("<I", "version")
    if version != 1:
        raise FormatError(f"unsupported version {version}", off - 4)
    kind = rd("<B", "cache kind")
    if kind > 1:
        raise FormatError(f"bad cache kind {kind}", off - 1)
    n = rd("<I", "stage count")
    if n < 1:
        raise FormatError("stage count must be >= 1", off - 4)
    stages = []
    for i in range(n):
        s = rd("<I", "codebook size")
        d = rd("<I", "dimension")
        if s < 1 or d < 1:
            raise FormatError("codebook size and dimension must be >= 1", off - 8)
        stage_off = off
        eb = inp.read(4 * s * d)
        if len(eb) != 4 * s * d:
            raise FormatError("truncated file reading entries", off)
        off += 4 * s * d
        pb = inp.read(4 * d * d)
        if len(pb) != 4 * d * d:
            raise FormatError("truncated file reading projection", off)
        off += 4 * d * d
        e = np.frombuffer(eb, np.float32).reshape(s, d).copy()
        p = np.frombuffer(pb, np.float32).reshape(d, d).copy()
        if not (np.isfinite(e).all() and np.isfinite(p).all()):
            raise FormatError(f"non-finite values in stage {i}", stage_off)
        stages.append(Codebook(e, p))
    st = CodebookStack(stages, kind, device)
    st.validate()
    _ = st.device  # refresh on load (codebook.cpp:312)
    return st


def stack_content_hash(stack: CodebookStack) -> int:
    """FNV-1a-64 over the serialized stack (codebook.cpp:326-336)."""
    buf = io.BytesIO()
    save_stack(stack, buf)
    h = 0xCBF29CE484222325
    for c in buf.getvalue():
        h ^= c
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h
