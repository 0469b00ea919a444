"""HCTRACE1 attention-trace container (host side, not on the hot path).

Same on-disk format, manifest keys, invariants and SHA-256 fingerprint as the
reference container (trace.py:1-391), so traces and reports are exchangeable
byte for byte with the reference package:

    "HCTRACE1" | u32 manifest_len | manifest JSON (sorted keys, compact) |
    (T+1) x layers x heads x K records of (u32 token_index, f32 score)

The GPU engine consumes the index/score arrays directly (trace-driven
parity mode), and tensor-mode runs export their score rows in this format
 so the reference can replay them.
"""

from __future__ import annotations

import hashlib
import io
import json
import struct
from dataclasses import dataclass, fields
from pathlib import Path

import numpy as np

MAGIC = b"HCTRACE1"
PAD_INDEX = 0xFFFFFFFF
_REC = np.dtype([("index", "<u4"), ("score", "<f4")])


class TraceError(Exception):
    """Base trace error (trace.py:50)."""


class TraceInvariantError(TraceError):
    pass


class TraceFormatError(TraceError):
    pass


class BadMagicError(TraceFormatError):
    pass


class UnsupportedVersionError(TraceFormatError):
    pass


class TruncatedPayloadError(TraceFormatError):
    def __init__(self, message: str, byte_offset: int):
        super().__init__(f"{message} (at byte offset {byte_offset})")
        self.byte_offset = byte_offset


@dataclass(frozen=True)
class TraceManifest:
    model_name: str
    num_layers: int
    heads_per_layer: int
    prefill_len: int
    decode_steps: int
    trace_topk: int
    pool_kernel_used: int = 0
    bytes_per_kv_entry: int = 256

    def validate(self) -> None:
        checks = (
            (self.num_layers >= 1, "num_layers must be >= 1"),
            (self.heads_per_layer >= 1, "heads_per_layer must be >= 1"),
            (self.prefill_len >= 1, "prefill_len must be >= 1"),
            (self.decode_steps >= 0, "decode_steps must be >= 0"),
            (self.trace_topk >= 1, "trace_topk must be >= 1"),
            (self.trace_topk <= self.prefill_len + self.decode_steps,
             "trace_topk must not exceed prefill_len + decode_steps"),
            (self.pool_kernel_used >= 0 and (self.pool_kernel_used == 0 or self.pool_kernel_used % 2),
             "pool_kernel_used must be odd or 0"),
            (self.bytes_per_kv_entry >= 1, "bytes_per_kv_entry must be >= 1"),
        )
        for ok, msg in checks:
            if not ok:
                raise TraceInvariantError(msg)

    def to_json_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    @classmethod
    def from_json_dict(cls, payload: dict) -> "TraceManifest":
        names = {f.name for f in fields(cls)}
        if set(payload) != names:
            raise TraceFormatError(
                f"manifest keys mismatch: missing={sorted(names - set(payload))} "
                f"extra={sorted(set(payload) - names)}")
        if not isinstance(payload["model_name"], str):
            raise TraceFormatError("manifest model_name must be a string")
        for n in names - {"model_name"}:
            v = payload[n]
            if not isinstance(v, int) or isinstance(v, bool):
                raise TraceFormatError(f"manifest {n} must be an integer")
        return cls(**payload)


@dataclass(frozen=True)
class AttentionTrace:
    manifest: TraceManifest
    indices: np.ndarray  # (T+1, layers, heads, K) uint32
    scores: np.ndarray   # (T+1, layers, heads, K) float32

    @property
    def num_steps(self) -> int:
        return self.manifest.decode_steps + 1

    def head_ids(self):
        m = self.manifest
        return [(l, h) for l in range(m.num_layers) for h in range(m.heads_per_layer)]


def _shape(m: TraceManifest):
    return (m.decode_steps + 1, m.num_layers, m.heads_per_layer, m.trace_topk)


def validate_trace(trace) -> None:
    """Invariants of trace.py:240-281."""
    m = trace.manifest
    m.validate()
    idx, sc = trace.indices, trace.scores
    if idx.shape != _shape(m) or sc.shape != _shape(m):
        raise TraceInvariantError(f"trace arrays must have shape {_shape(m)}")
    pad = idx == PAD_INDEX
    if (sc < 0).any():
        raise TraceInvariantError("scores must be nonnegative")
    if (sc[pad] != 0).any():
        raise TraceInvariantError("padding pairs must carry score 0.0")
    if m.trace_topk > 1:
        if (pad[..., :-1] & ~pad[..., 1:]).any():
            raise TraceInvariantError("padding pairs must form a suffix")
        if ((sc[..., :-1] < sc[..., 1:]) & ~pad[..., 1:]).any():
            raise TraceInvariantError("scores must be nonincreasing within a head")
    limit = (m.prefill_len + np.arange(m.decode_steps + 1, dtype=np.int64))[:, None, None, None]
    if ((idx.astype(np.int64) >= limit) & ~pad).any():
        raise TraceInvariantError("token index beyond sequence length")
    srt = np.sort(np.where(pad, -1, idx.astype(np.int64)), axis=-1)
    if ((srt[..., 1:] == srt[..., :-1]) & (srt[..., 1:] >= 0)).any():
        raise TraceInvariantError("duplicate token index")


def make_trace(manifest: TraceManifest, indices, scores) -> AttentionTrace:
    idx = np.ascontiguousarray(indices, dtype=np.uint32)
    sc = np.ascontiguousarray(scores, dtype=np.float32)
    if idx.shape != _shape(manifest) or sc.shape != _shape(manifest):
        raise TraceInvariantError(f"trace arrays must have shape {_shape(manifest)}")
    idx.setflags(write=False)
    sc.setflags(write=False)
    t = AttentionTrace(manifest, idx, sc)
    validate_trace(t)
    return t


def _manifest_bytes(m: TraceManifest) -> bytes:
    return json.dumps(m.to_json_dict(), sort_keys=True, separators=(",", ":")).encode()


def trace_bytes(trace) -> bytes:
    validate_trace(trace)
    body = np.empty(trace.indices.shape, dtype=_REC)
    body["index"] = trace.indices
    body["score"] = trace.scores
    mb = _manifest_bytes(trace.manifest)
    return MAGIC + struct.pack("<I", len(mb)) + mb + body.tobytes()


def write_trace(trace, destination) -> int:
    payload = trace_bytes(trace)
    if isinstance(destination, (str, Path)):
        p = Path(destination)
        tmp = p.with_name(p.name + ".tmp")
        tmp.write_bytes(payload)
        tmp.replace(p)
    else:
        destination.write(payload)
    return len(payload)


def read_trace(source) -> AttentionTrace:
    if isinstance(source, (str, Path)):
        data = Path(source).read_bytes()
    elif isinstance(source, (bytes, bytearray)):
        data = bytes(source)
    else:
        data = source.read()
    buf = io.BytesIO(data)

    def take(n, what, off):
        b = buf.read(n)
        if len(b) < n:
            raise TruncatedPayloadError(f"stream ended while reading {what}", off + len(b))
        return b

    magic = take(8, "magic", 0)
    if magic[:7] != MAGIC[:7]:
        raise BadMagicError(f"bad magic {magic!r}")
    if magic != MAGIC:
        raise UnsupportedVersionError(f"unsupported trace version {magic[7:]!r}")
    (mlen,) = struct.unpack("<I", take(4, "manifest length", 8))
    raw = take(mlen, "manifest", 12)
    try:
        obj = json.loads(raw.decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise TraceFormatError(f"manifest is not valid UTF-8 JSON: {exc}") from exc
    if not isinstance(obj, dict):
        raise TraceFormatError("manifest must be a JSON object")
    m = TraceManifest.from_json_dict(obj)
    m.validate()
    shape = _shape(m)
    nbytes = int(np.prod(shape)) * _REC.itemsize
    body = take(nbytes, "step records", 12 + mlen)
    if buf.read(1):
        raise TraceFormatError("trailing bytes after the final step record")
    rec = np.frombuffer(body, dtype=_REC).reshape(shape)
    return make_trace(m, rec["index"].copy(), rec["score"].copy())


def trace_fingerprint(trace) -> str:
    """trace.py:381-391: sha256(manifest JSON with default separators, idx, scores)."""
    h = hashlib.sha256()
    h.update(json.dumps(trace.manifest.to_json_dict(), sort_keys=True).encode())
    h.update(np.ascontiguousarray(trace.indices).tobytes())
    h.update(np.ascontiguousarray(trace.scores).tobytes())
    return h.hexdigest()
