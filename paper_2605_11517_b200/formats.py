"""On-disk formats shared with the reference (grinder/formats.py).

Little-endian, byte-identical to the reference writers:
  GRIN CSR   b"GRIN", u32 version=1, u64 |V|, u64 |E|, u64 src_ptr[|V|+1], u32 dst_idx[|E|]
  features   u64 rows, u64 cols, f32 row-major data
  u32 array  u64 count, u32 values
  checkpoint u64 L, u64 dims[L+1], f64 weight matrices
The readers memory-map the payload so multi-GB tier files load without an
extra copy.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .graph import CsrGraph

__all__ = ["CSR_MAGIC", "CSR_VERSION", "read_checkpoint", "read_csr_binary", "read_features",
           "read_u32_array", "write_checkpoint", "write_csr_binary", "write_features",
           "write_u32_array"]

CSR_MAGIC = b"GRIN"
CSR_VERSION = 1
_CSR_HEAD = struct.Struct("<4sIQQ")


def write_csr_binary(graph: CsrGraph, path: str | Path) -> None:
    with open(path, "wb") as fh:
        fh.write(_CSR_HEAD.pack(CSR_MAGIC, CSR_VERSION, graph.num_vertices, graph.num_edges))
        fh.write(np.ascontiguousarray(graph.src_ptr, dtype="<u8").tobytes())
        fh.write(np.ascontiguousarray(graph.dst_idx, dtype="<u4").tobytes())


def read_csr_binary(path: str | Path) -> CsrGraph:
    raw = np.memmap(path, dtype=np.uint8, mode="r")
    if raw.size < _CSR_HEAD.size or bytes(raw[:4]) != CSR_MAGIC:
        raise ValueError(f"not a CSR graph file: {path}")
    _, version, n, m = _CSR_HEAD.unpack(bytes(raw[:_CSR_HEAD.size]))
    if version != CSR_VERSION:
        raise ValueError(f"unsupported CSR version {version}")
    need = _CSR_HEAD.size + 8 * (n + 1) + 4 * m
    if raw.size != need:
        raise ValueError(f"truncated CSR file: expected {need} bytes, found {raw.size}")
    off = _CSR_HEAD.size
    ptr = np.frombuffer(raw, dtype="<u8", count=n + 1, offset=off).astype(np.int64)
    dst = np.frombuffer(raw, dtype="<u4", count=m, offset=off + 8 * (n + 1)).astype(np.int32)
    graph = CsrGraph(num_vertices=int(n), num_edges=int(m), src_ptr=ptr, dst_idx=dst)
    graph.validate()
    return graph


def write_features(path: str | Path, matrix: np.ndarray) -> None:
    mat = np.ascontiguousarray(matrix, dtype="<f4")
    if mat.ndim != 2:
        raise ValueError(f"feature matrix must be 2-D, got shape {matrix.shape}")
    with open(path, "wb") as fh:
        fh.write(struct.pack("<QQ", *mat.shape))
        fh.write(mat.tobytes())


def read_features(path: str | Path, dtype=np.float64, mmap: bool = False) -> np.ndarray:
    """Feature matrix as f64 (the reference's type) or, with dtype=float32,
    the stored values without conversion; ``mmap=True`` (float32 only)
    returns the memory-mapped rows themselves (no read), which the streaming
    engine serves from the file as its storage tier."""
    raw = np.memmap(path, dtype=np.uint8, mode="r")
    rows, cols = struct.unpack("<QQ", bytes(raw[:16]))
    need = 16 + 4 * rows * cols
    if raw.size != need:
        raise ValueError(f"truncated feature file: expected {need} bytes, found {raw.size}")
    vals = np.frombuffer(raw, dtype="<f4", count=rows * cols, offset=16).reshape(rows, cols)
    if mmap:
        if np.dtype(dtype) != np.float32:
            raise ValueError("mmap=True needs dtype=float32")
        return vals
    return vals.astype(dtype)


def write_u32_array(path: str | Path, values: np.ndarray) -> None:
    arr = np.asarray(values)
    if arr.ndim != 1:
        raise ValueError(f"expected a 1-D array, got shape {arr.shape}")
    if arr.size and (arr.min() < 0 or arr.max() > np.iinfo(np.uint32).max):
        raise ValueError("values out of u32 range")
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", arr.size))
        fh.write(arr.astype("<u4").tobytes())


def read_u32_array(path: str | Path) -> np.ndarray:
    raw = Path(path).read_bytes()
    (count,) = struct.unpack_from("<Q", raw, 0)
    if len(raw) != 8 + 4 * count:
        raise ValueError(f"truncated u32 array file: expected {8 + 4 * count} bytes, found {len(raw)}")
    return np.frombuffer(raw, dtype="<u4", count=count, offset=8).astype(np.int64)


def write_checkpoint(path: str | Path, weights: list[np.ndarray]) -> None:
    if not weights:
        raise ValueError("checkpoint requires at least one weight matrix")
    dims = [int(weights[0].shape[0])]
    for i, w in enumerate(weights):
        if w.ndim != 2:
            raise ValueError(f"weight {i} must be 2-D, got shape {w.shape}")
        if w.shape[0] != dims[-1]:
            raise ValueError(f"weight {i} input dim {w.shape[0]} != previous output {dims[-1]}")
        dims.append(int(w.shape[1]))
    with open(path, "wb") as fh:
        fh.write(struct.pack(f"<{len(dims) + 1}Q", len(weights), *dims))
        for w in weights:
            fh.write(np.ascontiguousarray(w, dtype="<f8").tobytes())


def read_checkpoint(path: str | Path) -> list[np.ndarray]:
    raw = Path(path).read_bytes()
    (layers,) = struct.unpack_from("<Q", raw, 0)
    dims = struct.unpack_from(f"<{layers + 1}Q", raw, 8)
    off = 8 * (layers + 2)
    out = []
    for r, c in zip(dims[:-1], dims[1:]):
        out.append(np.frombuffer(raw, dtype="<f8", count=r * c, offset=off).reshape(r, c).copy())
        off += 8 * r * c
    if off != len(raw):
        raise ValueError(f"trailing bytes in checkpoint: expected {off}, found {len(raw)}")
    return out


def canonical_json(obj) -> str:
    """JSON with sorted keys, 2-space indent and a trailing newline
    (formats.py:219-221): summaries and ledgers compare as text."""
    import json
    return json.dumps(obj, sort_keys=True, indent=2) + "\n"
