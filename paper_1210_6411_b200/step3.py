"""Paper-scale step 3 (SURVEY.md §8(d) C5, §5 checkpoint/resume): walk a start set in
chunks to per-chunk edge-record files, resumably.

The reference walks its skeleton with ``build_skeleton_edges`` (pipeline.py:231-256) in
one process and returns everything in memory; at paper scale (2^33.6 starts, 252 GB of
records) that is a multi-hour, multi-GPU job, so this driver keeps the
reference's record format and result but splits the work the way SPEC.md's manifest
describes (stage checkpoints with content digests):

* the start set (a ``uint64`` array, e.g. ``np.memmap`` of a ``write_states`` file) is cut
  into fixed chunks; rank ``r`` of ``world`` takes a contiguous run of chunks
  (``distributed.shard_range`` over the chunk count);
* each chunk is walked on the GPU (``walk_arrays`` -> K1) and written as one file of
  40-byte ``<5Q`` records (source, destination, distance, 0, 0) -- exactly the records
  ``build_skeleton_edges`` returns, in start order -- through a temporary name and an
  atomic rename;
* every finished chunk appends one JSON line to the rank's manifest (chunk range, file
  name, sha256 of the input states and of the file bytes, edge / transition counts,
  min / max distance), flushed and fsync'd;
* a rerun (``resume=True``) skips every chunk whose manifest line, file and digests still
  match, so an interrupted run continues where it stopped and a finished run is a no-op
  (SPEC.md's stage idempotence); a config mismatch with the manifest raises.

``merge_edge_files`` concatenates the chunk files in start order into one edge file (a
valid skeleton file when the starts were sorted, as step 1 emits them).
"""

from __future__ import annotations

import hashlib
import json
import os
from dataclasses import asdict, dataclass

import numpy as np

from . import records
from .bitslice import walk_arrays
from .cipher import CandidateParams, CipherSpec
from .distributed import shard_range

MANIFEST_VERSION = 1


@dataclass(frozen=True)
class ChunkRecord:
    index: int
    lo: int
    hi: int
    file: str
    input_sha256: str
    file_sha256: str
    edges: int
    transitions: int
    min_dist: int
    max_dist: int


def _sha256_file(path: str) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for blk in iter(lambda: f.read(1 << 24), b""):
            h.update(blk)
    return h.hexdigest()


def _config(spec: CipherSpec, params: CandidateParams, stride: int, chunk: int, n: int) -> dict:
    return {"version": MANIFEST_VERSION, "spec": json.loads(spec.to_json()), "fixed_r3": params.fixed_r3,
            "stride": int(stride), "chunk": int(chunk), "n": int(n)}


def _manifest_path(out_dir: str, rank: int) -> str:
    return os.path.join(out_dir, f"manifest.rank{rank}.jsonl")


def read_manifest(out_dir: str, rank: int = 0):
    """(config, {chunk index: ChunkRecord}) of one rank's manifest, or (None, {})."""
    path = _manifest_path(out_dir, rank)
    if not os.path.exists(path):
        return None, {}
    cfg, done = None, {}
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line:
                continue
            try:
                obj = json.loads(line)
            except json.JSONDecodeError:  # a torn last line after a crash: ignore it
                continue
            if obj.get("kind") == "config":
                cfg = obj["config"]
            elif obj.get("kind") == "chunk":
                rec = ChunkRecord(**obj["chunk"])
                done[rec.index] = rec
    return cfg, done


def _fsync_dir(path: str) -> None:
    """Make a rename in ``path`` durable (POSIX: the directory entry lives in the directory)."""
    try:
        fd = os.open(path, os.O_RDONLY)
    except OSError:
        return
    try:
        os.fsync(fd)
    except OSError:
        pass
    finally:
        os.close(fd)


def _append(path: str, obj: dict) -> None:
    with open(path, "a") as f:
        f.write(json.dumps(obj) + "\n")
        f.flush()
        os.fsync(f.fileno())


def walk_to_edge_files(states, out_dir: str, spec: CipherSpec, params: CandidateParams, *, stride: int,
                       chunk: int = 1 << 24, rank: int = 0, world: int = 1, resume: bool = True,
                       max_clocks: int | None = None) -> list:
    """Walk this rank's chunks of ``states`` (bitslice.forward_to_candidate semantics, one
    hop at ``stride``) into ``out_dir``; returns the rank's ChunkRecords in chunk order
    (resumed ones included)."""
    states = np.asarray(states)
    if states.dtype != np.uint64 or states.ndim != 1:
        raise ValueError("states must be a 1-D uint64 array")
    if chunk < 1:
        raise ValueError("chunk must be >= 1")
    n = int(states.size)
    os.makedirs(out_dir, exist_ok=True)
    cfg = _config(spec, params, stride, chunk, n)
    mpath = _manifest_path(out_dir, rank)
    old_cfg, done = read_manifest(out_dir, rank) if resume else (None, {})
    if old_cfg is not None and old_cfg != cfg:
        raise ValueError(f"{mpath} was written for another configuration: {old_cfg} != {cfg}")
    if old_cfg is None or not resume:
        if os.path.exists(mpath):
            os.remove(mpath)
        _append(mpath, {"kind": "config", "config": cfg})
        done = {}
    n_chunks = (n + chunk - 1) // chunk
    c_lo, c_hi = shard_range(n_chunks, rank, world)
    out = []
    for c in range(c_lo, c_hi):
        lo, hi = c * chunk, min(n, (c + 1) * chunk)
        part = np.ascontiguousarray(states[lo:hi])
        in_sha = hashlib.sha256(part.astype("<u8", copy=False).tobytes()).hexdigest()
        name = f"edges_{lo:012d}_{hi:012d}.bin"
        path = os.path.join(out_dir, name)
        rec = done.get(c)
        if (rec is not None and rec.input_sha256 == in_sha and rec.file == name and os.path.exists(path)
                and os.path.getsize(path) == (hi - lo) * records.EDGE_SIZE and _sha256_file(path) == rec.file_sha256):
            out.append(rec)
            continue
        res = walk_arrays(part, params, spec, stride=stride, max_clocks=max_clocks)
        dst, dist = res.dst[:, 0], res.dist[:, 0]
        tmp = path + ".tmp"
        records.write_edge_arrays(tmp, part, dst, dist)
        with open(tmp, "rb+") as f:
            os.fsync(f.fileno())
        os.replace(tmp, path)
        _fsync_dir(out_dir)
        rec = ChunkRecord(index=c, lo=lo, hi=hi, file=name, input_sha256=in_sha, file_sha256=_sha256_file(path),
                          edges=int(res.edges), transitions=int(res.transitions),
                          min_dist=int(dist.min()) if dist.size else 0, max_dist=int(dist.max()) if dist.size else 0)
        _append(mpath, {"kind": "chunk", "chunk": asdict(rec)})
        out.append(rec)
    return out


def merge_edge_files(out_dir: str, out_path: str, ranks: int = 1) -> int:
    """Concatenate every rank's chunk files in start order into one edge file; returns the
    record count.  Raises if a chunk is missing or its bytes changed."""
    recs, n = [], None
    for r in range(ranks):
        cfg, done = read_manifest(out_dir, r)
        if cfg is None:
            raise ValueError(f"no manifest for rank {r} in {out_dir}")
        if n is not None and cfg["n"] != n:
            raise ValueError("the ranks' manifests describe different start sets")
        n = cfg["n"]
        recs.extend(done.values())
    recs.sort(key=lambda x: x.lo)
    pos = 0
    for rec in recs:
        if rec.lo != pos:
            raise ValueError(f"chunk starting at {pos} is missing" if rec.lo > pos
                             else f"chunk starting at {rec.lo} is listed twice")
        pos = rec.hi
    if pos != n:
        raise ValueError(f"chunks after record {pos} of {n} are missing")
    total = 0
    tmp = out_path + ".tmp"
    with open(tmp, "wb") as w:
        for rec in recs:
            path = os.path.join(out_dir, rec.file)
            if _sha256_file(path) != rec.file_sha256:
                raise ValueError(f"{path} does not match its manifest digest")
            with open(path, "rb") as f:
                for blk in iter(lambda: f.read(1 << 24), b""):
                    w.write(blk)
            total += rec.hi - rec.lo
    os.replace(tmp, out_path)
    _fsync_dir(os.path.dirname(os.path.abspath(out_path)))
    return total
