"""Device-resident blocked compressed-sparse-column (BCSC) matrices.

Mirrors ``blocksparse.bcsc`` (pkg/src/blocksparse/bcsc.py) with the arrays in
HBM:

* ``col_ptr``        int64 [grid_cols + 1]   (bcsc.py:42-43)
* ``block_row_idx``  int32 [nnzb]            (uint32 in the reference; same values)
* ``values``         [nnzb, b, b] float32 or bfloat16, row-major inside a block,
  ``values[k][i][j] = W[r*b + i, c*b + j]`` (bcsc.py:46-47, :199, :210)

plus ``kmap`` [grid_rows, grid_cols] int32 (stored block index or -1), from
which the kernels' execution plans are derived (csrc/plan.cu). Conversion
(``from_dense``) runs on the GPU (csrc/prune.cu repack kernels). Matrices are
immutable after construction, like the reference (bcsc.py:35).

The binary ``BCSC`` v1 serialization (bcsc.py:17-20, :233-289) is byte
identical to the reference's so checkpoints interoperate.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _arrays as A
from . import _lib as L

MAGIC = b"BCSC"
FORMAT_VERSION = 1
_HEADER = struct.Struct("<4sIQQIQ")  # magic, version, rows, cols, block, nnzb
DENSE_MAGIC = b"DNSE"
_DENSE_HEADER = struct.Struct("<4sIII")


class FormatError(ValueError):
    """Raised when a serialized matrix stream is malformed (bcsc.py:27-28)."""


def _grid_dim(n: int, b: int) -> int:
    return -(-n // b)


@dataclass(eq=False)
class BlockSparseMatrix:
    rows: int
    cols: int
    block: int
    col_ptr: torch.Tensor
    block_row_idx: torch.Tensor
    values: torch.Tensor
    kmap: torch.Tensor | None = None
    host_api: bool = False
    _cache: dict = field(default_factory=dict, repr=False)

    # ------------------------------------------------------------ shape
    @property
    def grid_rows(self) -> int:
        return _grid_dim(self.rows, self.block)

    @property
    def grid_cols(self) -> int:
        return _grid_dim(self.cols, self.block)

    @property
    def nnzb(self) -> int:
        return int(self.block_row_idx.shape[0])

    @property
    def dtype(self) -> torch.dtype:
        return self.values.dtype

    def to_dense(self):
        return to_dense(self)

    def block_sparsity(self) -> float:
        return block_sparsity(self)

    # ------------------------------------------------------------ device plumbing
    def _kmap(self) -> torch.Tensor:
        if self.kmap is None:
            km = torch.empty(self.grid_rows, self.grid_cols, dtype=torch.int32, device=A.DEVICE)
            L.check(L.load().blast_kmap_from_bcsc(
                self.col_ptr.data_ptr(), self.block_row_idx.data_ptr() if self.nnzb else None,
                self.grid_rows, self.grid_cols, km.data_ptr(), L.stream()), "kmap")
            self.kmap = km
        return self.kmap

    def _plan(self, by_rows: int):
        key = ("plan", by_rows)
        if key not in self._cache:
            self._cache[key] = build_plan(self._kmap(), None, self.grid_rows, self.grid_cols,
                                          by_rows)
        return self._cache[key]

    def wgrad_plan(self):
        """(items, counts) of the stored-block weight-gradient work list (blast_wgrad_plan),
        cached with the structure like the product plans; None when b is not 64 / 128."""
        if self.block not in (64, 128) or self.nnzb == 0:
            return None
        if "wgrad" not in self._cache:
            items = torch.empty(self.nnzb, 4, dtype=torch.int32, device=A.DEVICE)
            counts = torch.empty(self.grid_cols + 1, dtype=torch.int64, device=A.DEVICE)
            L.check(L.load().blast_wgrad_plan(self.col_ptr.data_ptr(), self.grid_rows,
                                              self.grid_cols, self.block, items.data_ptr(),
                                              counts.data_ptr(), L.stream()), "wgrad_plan")
            self._cache["wgrad"] = (items, counts)
        return self._cache["wgrad"]

    def _tf32(self):
        """hi/lo tf32 images of the float32 blocks (3xTF32 operands). They are derived
        data: re-split in place whenever ``values`` was modified since the last split
        (tracked by the tensor's version counter, which in-place optimizer steps and
        ``load_state_dict`` bump), so the tensor-core path never reads stale weights."""
        v = self.values
        if v.dtype != torch.float32:
            raise ValueError("3xTF32 operands only exist for float32 matrices")
        parts = self._cache.get("tf32")
        if parts is None:
            parts = [torch.empty_like(v) for _ in range(4)]
            self._cache["tf32"] = parts
            self._cache["tf32_version"] = None
        ver = (v.data_ptr(), v._version)
        if self._cache["tf32_version"] != ver:
            if self.nnzb:
                L.check(L.load().blast_tf32_prepare(v.data_ptr(), self.nnzb, self.block,
                                                    *[p.data_ptr() for p in parts], L.stream()),
                        "tf32_prepare")
            self._cache["tf32_version"] = ver
        return parts

    def desc(self) -> L.BcscDesc:
        """C descriptor (include/blast.h blast_bcsc_t) with plans built on first use.
        The descriptor is rebuilt if ``values`` was rebound to other storage, and the
        3xTF32 images are refreshed when the values changed in place."""
        d = self._cache.get("desc")
        if d is not None and self._cache.get("desc_values") == self.values.data_ptr():
            if self.values.dtype == torch.float32:
                self._tf32()
            return d
        fwd = self._plan(0)
        rt = self._plan(1)
        tf = self._tf32() if self.values.dtype == torch.float32 else [None] * 4
        d = L.BcscDesc(
            self.rows, self.cols, self.block, L.dtype_code(self.values.dtype), self.nnzb,
            self.col_ptr.data_ptr(), self.block_row_idx.data_ptr() if self.nnzb else None,
            self.values.data_ptr() if self.nnzb else None,
            *[L.ptr(t) if self.nnzb else None for t in tf],
            self._kmap().data_ptr(),
            fwd[0].data_ptr(), fwd[1].data_ptr(), fwd[2].data_ptr(),
            rt[0].data_ptr(), rt[1].data_ptr(), rt[2].data_ptr(),
        )
        self._cache["desc"] = d
        self._cache["desc_values"] = self.values.data_ptr()
        return d

    # ------------------------------------------------------------ host views
    def to_host(self) -> "HostBCSC":
        """numpy copy with the reference's dtypes (int64 / uint32 / float32)."""
        return HostBCSC(
            rows=self.rows, cols=self.cols, block=self.block,
            col_ptr=self.col_ptr.cpu().numpy().astype(np.int64),
            block_row_idx=self.block_row_idx.cpu().numpy().astype(np.uint32),
            values=A.to_host(self.values).astype(np.float32).reshape(self.nnzb, self.block,
                                                                     self.block),
        )

    def astype(self, dtype: torch.dtype) -> "BlockSparseMatrix":
        if dtype == self.values.dtype:
            return self
        return BlockSparseMatrix(self.rows, self.cols, self.block, self.col_ptr,
                                 self.block_row_idx, self.values.to(dtype).contiguous(),
                                 self.kmap, self.host_api)

    def validate(self) -> None:
        """Structural invariants (bcsc.py:75-109), checked on a host copy."""
        h = self.to_host()
        gr, gc, b = self.grid_rows, self.grid_cols, self.block
        if b < 1:
            raise ValueError("block size must be >= 1")
        if h.col_ptr.shape != (gc + 1,):
            raise ValueError(f"col_ptr length {h.col_ptr.shape[0]} != grid_cols+1 ({gc + 1})")
        if h.col_ptr[0] != 0 or h.col_ptr[-1] != self.nnzb:
            raise ValueError("col_ptr must start at 0 and end at nnzb")
        if np.any(np.diff(h.col_ptr) < 0):
            raise ValueError("col_ptr must be nondecreasing")
        if h.values.shape != (self.nnzb, b, b):
            raise ValueError(f"values shape {h.values.shape} != (nnzb, b, b)")
        if self.nnzb and int(h.block_row_idx.max()) >= gr:
            raise ValueError("block row index out of range")
        cols_of = np.repeat(np.arange(gc), np.diff(h.col_ptr))
        if self.nnzb > 1:
            same = cols_of[1:] == cols_of[:-1]
            if np.any(np.diff(h.block_row_idx.astype(np.int64))[same] <= 0):
                raise ValueError("block rows not strictly increasing within a column")
        pad_r, pad_c = gr * b - self.rows, gc * b - self.cols
        if pad_r and np.any(h.values[h.block_row_idx == gr - 1][:, b - pad_r:, :]):
            raise ValueError("nonzero values in row padding region")
        if pad_c and np.any(h.values[cols_of == gc - 1][:, :, b - pad_c:]):
            raise ValueError("nonzero values in column padding region")


@dataclass(frozen=True)
class HostBCSC:
    """Reference-layout numpy snapshot of a device matrix."""
    rows: int
    cols: int
    block: int
    col_ptr: np.ndarray
    block_row_idx: np.ndarray
    values: np.ndarray

    @property
    def nnzb(self) -> int:
        return int(self.block_row_idx.shape[0])


def build_plan(kmap0: torch.Tensor, kmap1: torch.Tensor | None, gr: int, gc: int, by_rows: int):
    lines = gr if by_rows else gc
    step_ptr = torch.empty(lines + 1, dtype=torch.int32, device=A.DEVICE)
    steps = torch.empty(max(gr * gc, 1) * 4, dtype=torch.int32, device=A.DEVICE)
    flags = torch.empty(max(lines, 1), dtype=torch.int32, device=A.DEVICE)
    L.check(L.load().blast_build_plan(kmap0.data_ptr(), L.ptr(kmap1), gr, gc, by_rows,
                                      step_ptr.data_ptr(), steps.data_ptr(), flags.data_ptr(),
                                      L.stream()), "build_plan")
    return step_ptr, steps, flags


@dataclass(frozen=True)
class BlockMask:
    """kept / regrown block grids (bcsc.py:112-156). Arrays are numpy bool grids for
    host callers or CUDA bool tensors for device callers."""
    kept: object
    regrown: object
    # (|kept|, |regrown|) when known from the kernels that built the mask (generate_masks):
    # lets apply_mask size the repack without reading nnzb back from the device
    counts: tuple | None = field(default=None, compare=False, repr=False)

    @classmethod
    def trusted(cls, kept, regrown, n_kept: int, n_regrown: int) -> "BlockMask":
        """Mask from grids that are disjoint by construction (device bool grids of
        generate_masks): skips the validation pass and its host synchronisation."""
        m = object.__new__(cls)
        object.__setattr__(m, "kept", kept)
        object.__setattr__(m, "regrown", regrown)
        object.__setattr__(m, "counts", (int(n_kept), int(n_regrown)))
        return m

    @property
    def known_active(self) -> int | None:
        return None if self.counts is None else self.counts[0] + self.counts[1]

    def __post_init__(self):
        if A.shape(self.kept) != A.shape(self.regrown):
            raise ValueError("kept and regrown grids must have the same shape")
        if A.ndim(self.kept) != 2:
            raise ValueError("mask grids must be 2-D")
        if isinstance(self.kept, torch.Tensor):
            if bool((self.kept.bool() & self.regrown.bool()).any()):
                raise ValueError("kept and regrown must be disjoint")
        elif np.any(np.asarray(self.kept) & np.asarray(self.regrown)):
            raise ValueError("kept and regrown must be disjoint")

    @property
    def grid_rows(self) -> int:
        return A.shape(self.kept)[0]

    @property
    def grid_cols(self) -> int:
        return A.shape(self.kept)[1]

    @property
    def active(self):
        if isinstance(self.kept, torch.Tensor):
            return self.kept.bool() | self.regrown.bool()
        return np.asarray(self.kept) | np.asarray(self.regrown)

    @property
    def n_active(self) -> int:
        if self.counts is not None:
            return self.counts[0] + self.counts[1]
        a = self.active
        return int(a.sum().item()) if isinstance(a, torch.Tensor) else int(np.count_nonzero(a))

    def block_sparsity(self) -> float:
        return 1.0 - self.n_active / (self.grid_rows * self.grid_cols)

    def device_u8(self):
        """(kept, regrown) as contiguous uint8 CUDA grids for the kernels."""
        def u8(g):
            t = A.to_device(g)
            if t.dtype == torch.bool and t.is_contiguous():
                return t.view(torch.uint8)  # same bytes (0 / 1), no conversion kernel
            return t.to(torch.uint8).contiguous()
        return u8(self.kept), u8(self.regrown)

    @classmethod
    def all_active(cls, grid_rows: int, grid_cols: int, device: bool = False) -> "BlockMask":
        if device:
            return cls(kept=torch.ones(grid_rows, grid_cols, dtype=torch.bool, device=A.DEVICE),
                       regrown=torch.zeros(grid_rows, grid_cols, dtype=torch.bool,
                                           device=A.DEVICE))
        return cls(kept=np.ones((grid_rows, grid_cols), dtype=bool),
                   regrown=np.zeros((grid_rows, grid_cols), dtype=bool))


def expand_mask(grid, b: int, rows: int, cols: int):
    """Block grid -> element grid (rows x cols), same array kind as the input."""
    if isinstance(grid, torch.Tensor):
        return grid.repeat_interleave(b, 0).repeat_interleave(b, 1)[:rows, :cols]
    g = np.asarray(grid)
    return np.repeat(np.repeat(g, b, axis=0), b, axis=1)[:rows, :cols]


def _check_dense(dense, b: int):
    if A.ndim(dense) != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={A.ndim(dense)}")
    rows, cols = A.shape(dense)
    if rows < 1 or cols < 1:
        raise ValueError(f"matrix dimensions must be positive, got {(rows, cols)}")
    if b < 1:
        raise ValueError(f"block size must be >= 1, got {b}")
    return rows, cols


def _repack(dense_t: torch.Tensor, b: int, kept_u8, regrown_u8, values_dtype: torch.dtype,
            nnzb: int | None = None):
    """Index pass of the repack: col_ptr + kmap on device. ``nnzb`` (the active-block count,
    known after generate_masks) sizes the outputs without a host round trip; otherwise it is
    read back from col_ptr (one D2H sync)."""
    lib = L.load()
    rows, cols = dense_t.shape
    gr, gc = _grid_dim(rows, b), _grid_dim(cols, b)
    col_ptr = torch.empty(gc + 1, dtype=torch.int64, device=A.DEVICE)
    kmap = torch.empty(gr, gc, dtype=torch.int32, device=A.DEVICE)
    L.check(lib.blast_repack_index(L.ptr(kept_u8), L.ptr(regrown_u8), dense_t.data_ptr(), rows,
                                   cols, b, L.dtype_code(dense_t.dtype), col_ptr.data_ptr(),
                                   kmap.data_ptr(), L.stream()), "repack_index")
    if nnzb is None:
        nnzb = int(col_ptr[-1].item())
    row_idx = torch.empty(nnzb, dtype=torch.int32, device=A.DEVICE)
    if nnzb:
        L.check(lib.blast_repack_rows(kmap.data_ptr(), col_ptr.data_ptr(), gr, gc,
                                      row_idx.data_ptr(), L.stream()), "repack_rows")
    padded = rows % b != 0 or cols % b != 0
    alloc = torch.zeros if padded else torch.empty
    values = alloc((nnzb, b, b), dtype=values_dtype, device=A.DEVICE)
    return col_ptr, row_idx, kmap, values


def from_dense(dense, b: int, mask: BlockMask | None = None,
               dtype: torch.dtype | None = None) -> BlockSparseMatrix:
    """Dense -> BCSC on the GPU (bcsc.py:175-214).

    Without a mask every block holding a nonzero entry is stored; with a mask
    exactly the active blocks are stored, values copied verbatim (zeros too).
    ``dtype`` selects the stored value type (default: float32, or bfloat16 for
    bf16 input tensors).
    """
    rows, cols = _check_dense(dense, b)
    gr, gc = _grid_dim(rows, b), _grid_dim(cols, b)
    if mask is not None and (mask.grid_rows, mask.grid_cols) != (gr, gc):
        raise ValueError(
            f"mask grid {mask.grid_rows}x{mask.grid_cols} does not match "
            f"matrix grid {gr}x{gc} for block size {b}")
    host = A.is_host(dense)
    dense_t = A.to_device(dense, A.float_dtype(dense))
    vdt = dtype or dense_t.dtype
    kept, regrown = mask.device_u8() if mask is not None else (None, None)
    col_ptr, row_idx, kmap, values = _repack(dense_t, b, kept, regrown, vdt)
    if values.numel():
        L.check(L.load().blast_apply_mask_gather(
            dense_t.data_ptr(), rows, cols, b, L.dtype_code(dense_t.dtype), None, None, 0,
            kmap.data_ptr(), None, values.data_ptr(), L.dtype_code(vdt), L.stream()), "gather")
    return BlockSparseMatrix(rows, cols, b, col_ptr, row_idx, values, kmap, host)


def from_host(w, dtype: torch.dtype = torch.float32) -> BlockSparseMatrix:
    """Upload a reference-layout matrix (anything with rows/cols/block/col_ptr/
    block_row_idx/values, e.g. a ``blocksparse.bcsc.BlockSparseMatrix``)."""
    vals = torch.from_numpy(np.ascontiguousarray(np.asarray(w.values, dtype=np.float32)))
    return BlockSparseMatrix(
        int(w.rows), int(w.cols), int(w.block),
        torch.from_numpy(np.asarray(w.col_ptr, dtype=np.int64)).to(A.DEVICE),
        torch.from_numpy(np.asarray(w.block_row_idx).astype(np.int32)).to(A.DEVICE),
        vals.to(A.DEVICE).to(dtype).contiguous(), None, True)


def to_dense(w: BlockSparseMatrix):
    """Logical dense matrix; absent blocks are zero (bcsc.py:217-225)."""
    b, gr, gc = w.block, w.grid_rows, w.grid_cols
    out = torch.zeros(gr * gc, b, b, dtype=w.values.dtype, device=A.DEVICE)
    if w.nnzb:
        km = w._kmap().reshape(-1).long()
        present = km >= 0
        out[present] = w.values[km[present]]
    dense = out.reshape(gr, gc, b, b).permute(0, 2, 1, 3).reshape(gr * b, gc * b)
    dense = dense[: w.rows, : w.cols].contiguous()
    return A.like_input(dense, w.host_api)


def block_sparsity(w: BlockSparseMatrix) -> float:
    return 1.0 - w.nnzb / (w.grid_rows * w.grid_cols)


# ---------------------------------------------------------------- serialization
def serialize(w: BlockSparseMatrix) -> bytes:
    """Little-endian ``BCSC`` v1 bytes, identical to bcsc.py:233-241 (values as f32)."""
    h = w.to_host()
    header = _HEADER.pack(MAGIC, FORMAT_VERSION, h.rows, h.cols, h.block, h.nnzb)
    return b"".join((header, h.col_ptr.astype("<u8").tobytes(),
                     h.block_row_idx.astype("<u4").tobytes(), h.values.astype("<f4").tobytes()))


def deserialize(data: bytes, dtype: torch.dtype = torch.float32) -> BlockSparseMatrix:
    if len(data) < _HEADER.size:
        raise FormatError("truncated stream: incomplete header")
    magic, version, rows, cols, block, nnzb = _HEADER.unpack_from(data)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if version != FORMAT_VERSION:
        raise FormatError(f"unsupported format version {version}")
    if block < 1 or rows < 1 or cols < 1:
        raise FormatError("invalid header dimensions")
    gc = _grid_dim(cols, block)
    need = _HEADER.size + (gc + 1) * 8 + nnzb * 4 + nnzb * block * block * 4
    if len(data) < need:
        raise FormatError(f"truncated stream: expected {need} bytes, got {len(data)}")
    if len(data) > need:
        raise FormatError(f"trailing data: expected {need} bytes, got {len(data)}")
    off = _HEADER.size
    col_ptr = np.frombuffer(data, "<u8", gc + 1, off).astype(np.int64)
    off += (gc + 1) * 8
    rows_idx = np.frombuffer(data, "<u4", nnzb, off).astype(np.uint32)
    off += nnzb * 4
    vals = np.frombuffer(data, "<f4", nnzb * block * block, off).reshape(nnzb, block, block)
    host = HostBCSC(rows, cols, block, col_ptr, rows_idx, vals.astype(np.float32))
    w = from_host(host, dtype)
    try:
        w.validate()
    except ValueError as exc:
        raise FormatError(f"invariant violation after load: {exc}") from exc
    return w


def save(w: BlockSparseMatrix, path) -> None:
    with open(path, "wb") as fh:
        fh.write(serialize(w))


def load(path, dtype: torch.dtype = torch.float32) -> BlockSparseMatrix:
    with open(path, "rb") as fh:
        return deserialize(fh.read(), dtype)


def write_dense_file(dense, path) -> None:
    """Dense float32 matrix in the raw little-endian ``DNSE`` interchange format
    (header magic, rows, cols, 0; then row-major f32), as bcsc.py:292-300."""
    d = dense.detach().float().cpu().numpy() if isinstance(dense, torch.Tensor) else \
        np.asarray(dense, dtype=np.float32)
    if d.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    rows, cols = d.shape
    with open(path, "wb") as fh:
        fh.write(_DENSE_HEADER.pack(DENSE_MAGIC, rows, cols, 0))
        fh.write(np.ascontiguousarray(d).astype("<f4").tobytes())


def read_dense_file(path) -> np.ndarray:
    """Inverse of write_dense_file with the reference's checks (bcsc.py:303-314)."""
    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < _DENSE_HEADER.size:
        raise FormatError("truncated stream: incomplete dense header")
    magic, rows, cols, _ = _DENSE_HEADER.unpack_from(data)
    if magic != DENSE_MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {DENSE_MAGIC!r}")
    need = _DENSE_HEADER.size + rows * cols * 4
    if len(data) != need:
        raise FormatError(f"dense payload size mismatch: expected {need} bytes, got {len(data)}")
    return np.frombuffer(data, "<f4", rows * cols, _DENSE_HEADER.size).astype(np.float32).reshape(rows, cols)


def convert(input_path, output_path, block_size: int = 64):
    """The reference's ``convert`` command as a library call (cli.py:231-247): a ``DNSE``
    dense file becomes a ``BCSC`` file (every block holding a nonzero stored, repacked on the
    GPU), a ``BCSC`` file becomes a ``DNSE`` dense file. Returns the matrix written."""
    with open(input_path, "rb") as fh:
        magic = fh.read(4)
    if magic == DENSE_MAGIC:
        w = from_dense(read_dense_file(input_path), block_size)
        save(w, output_path)
        return w
    if magic == MAGIC:
        dense = to_dense(load(input_path))
        write_dense_file(dense, output_path)
        return dense
    raise FormatError(f"{input_path}: unrecognized magic {magic!r} (expected DNSE or BCSC)")
