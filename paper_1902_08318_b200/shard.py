"""Byte-range sharding of one document across GPUs (shard.h).

Shard g of G parses bytes [begin, end) of the document; four fixed-size
summaries are all-gathered between its phases.  `run_shard` drives one shard
with an `exchange(phase, local) -> gathered` callable:

  * `nccl_exchange(dist)`   one process per GPU: torch.distributed
                            all_gather_into_tensor (NCCL over NVLink);
  * `LocalShards`           G shards emulated in one process (one GPU): each
                            shard writes its summary straight into the
                            gathered buffer, phases run in lock step.

Results match jt_parse of the whole document: the same error code and
offset, and (on success) the document tape / string buffer is the
concatenation of the shards' parts (`assemble`).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .jsontape import ERROR_NAMES, Parser, load_library

TILE = 16384  # K1 tile (stage1.h kStage1Tile); shard starts are tile-aligned


def layout(length: int, shards: int) -> list[tuple[int, int]]:
    """Tile-aligned byte ranges [begin, end) covering [0, length), one per
    shard; every range is non-empty (so at most ceil(length / TILE) shards)."""
    tiles = max(1, (length + TILE - 1) // TILE)
    if shards < 1 or shards > tiles:
        raise ValueError(f"{shards} shards for {length} bytes ({tiles} tiles)")
    cuts = [(g * tiles // shards) * TILE for g in range(shards)] + [length]
    return [(cuts[g], min(cuts[g + 1], length)) for g in range(shards)]


def set_resident(parser: Parser, lo: int, hi: int):
    """Only bytes [lo, hi) of the document are on this parser's GPU (hi = 0:
    all).  A number of the shard running to hi fails the parse with
    CAPACITY (offset -1) instead of reading bytes that are not there."""
    lib = load_library()
    if lib.jt_b200_shard_resident(parser._h, lo, hi) != 0:
        raise RuntimeError(lib.jt_b200_last_error(parser._h).decode())


def summary_bytes(phase: int) -> int:
    return int(load_library().jt_b200_shard_summary_bytes(phase))


def _begin(parser: Parser, length: int, g: int, G: int):
    lib = load_library()
    b, e = layout(length, G)[g]
    if lib.jt_b200_shard_begin(parser._h, length, g, G, b, e) != 0:
        raise RuntimeError(lib.jt_b200_last_error(parser._h).decode())


def _phase(parser: Parser, k: int, gathered, out):
    lib = load_library()
    gp = 0 if gathered is None else gathered.data_ptr()
    if lib.jt_b200_shard_phase(parser._h, k, gp or None, out.data_ptr()) != 0:
        raise RuntimeError(lib.jt_b200_last_error(parser._h).decode())


def _finish(parser: Parser, gathered) -> tuple[str, int]:
    lib = load_library()
    off = C.c_longlong()
    code = lib.jt_b200_shard_finish(parser._h, gathered.data_ptr(), C.byref(off))
    return ERROR_NAMES[code], off.value


def run_shard(parser: Parser, length: int, g: int, G: int, exchange, device=None, mark=None):
    """Parse shard g of G of the `length` bytes resident in `parser`'s input
    buffer; `exchange(phase, local)` returns the G gathered summaries as one
    uint8 CUDA tensor.  Returns (error name, offset) for the whole document.
    `mark(phase)` (optional) is called after each phase's exchange."""
    import torch
    stream = torch.cuda.current_stream()
    if stream.cuda_stream == 0:
        raise RuntimeError("run_shard needs a non-default current stream (the legacy NULL "
                           "stream means 'the parser's own stream' in the C ABI)")
    parser.set_stream(stream.cuda_stream)
    _begin(parser, length, g, G)
    gathered = None
    for k in range(4):
        out = torch.empty(summary_bytes(k), dtype=torch.uint8, device=device or "cuda")
        _phase(parser, k, gathered, out)
        gathered = exchange(k, out)
        if mark:
            mark(k)
    return _finish(parser, gathered)


def nccl_exchange(dist, world: int):
    """all_gather of each phase's summary over the default process group."""
    import torch

    def ex(phase, local):
        out = torch.empty(world * local.numel(), dtype=torch.uint8, device=local.device)
        try:
            dist.all_gather_into_tensor(out, local)
        except (RuntimeError, NotImplementedError, AttributeError):  # backends without it
            parts = [torch.empty_like(local) for _ in range(world)]
            dist.all_gather(parts, local)
            out = torch.cat(parts)
        return out
    return ex


def host_exchange(dist, world: int):
    """The same all_gather staged through host memory (gloo: ranks that share
    one GPU, as the multi-process tests and bench.py's JT_BENCH_GLOO mode)."""
    import torch

    def ex(phase, local):
        h = local.cpu()
        parts = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(parts, h)
        return torch.cat(parts).to(local.device)
    return ex


class LocalShards:
    """G shards of one document on the current GPU (one parser each), phases
    in lock step on torch's current stream; the exchange is in-place: every
    shard writes its summary into its slot of the gathered buffer."""

    def __init__(self, data: bytes, G: int):
        import torch
        self.G = G
        self.len = len(data)
        self.parsers = [Parser() for _ in range(G)]
        # one real stream orders all shards' phases (torch's legacy default
        # stream would mean "each parser's own stream" in the C ABI)
        self.stream = torch.cuda.Stream()
        host = torch.frombuffer(bytearray(data), dtype=torch.uint8) if data else torch.zeros(1, dtype=torch.uint8)
        for p in self.parsers:
            p.set_stream(self.stream.cuda_stream)
            p.copy_in(host.data_ptr(), self.len)

    def run(self) -> tuple[str, int]:
        import torch
        with torch.cuda.stream(self.stream):
            return self._run()

    def _run(self) -> tuple[str, int]:
        import torch
        for g, p in enumerate(self.parsers):
            _begin(p, self.len, g, self.G)
        gathered = None
        for k in range(4):
            nb = summary_bytes(k)
            nxt = torch.empty(self.G * nb, dtype=torch.uint8, device="cuda")
            for g, p in enumerate(self.parsers):
                _phase(p, k, gathered, nxt[g * nb:(g + 1) * nb])
            gathered = nxt
        results = [_finish(p, gathered) for p in self.parsers]
        assert all(r == results[0] for r in results), results
        return results[0]

    def assemble(self) -> tuple[np.ndarray, bytes]:
        """Document tape and string buffer from the shards (after a successful run)."""
        return assemble(self.parsers)

    def close(self):
        for p in self.parsers:
            p.close()


def extent(parser: Parser) -> list[int]:
    out = (C.c_ulonglong * 7)()
    if load_library().jt_b200_shard_extent(parser._h, out) != 0:
        raise RuntimeError("no shard")
    return list(out)


def download(parser: Parser) -> tuple[int, np.ndarray, int, bytes]:
    """(document tape index, local tape words, document string offset, bytes)."""
    e = extent(parser)
    tape = np.zeros(max(1, e[2]), dtype=np.uint64)
    strings = C.create_string_buffer(max(1, e[4]))
    if load_library().jt_b200_shard_download(parser._h, tape.ctypes.data, strings) != 0:
        raise RuntimeError("shard download failed")
    return e[0], tape[:e[2]], e[3], strings.raw[:e[4]]


def assemble(parsers) -> tuple[np.ndarray, bytes]:
    parts = [download(p) for p in parsers]
    tape = np.concatenate([t for _, t, _, _ in parts])
    strings = b"".join(s for _, _, _, s in parts)
    at = 0
    for t0, t, s0, s in parts:
        assert t0 == at, (t0, at)
        at += len(t)
    return tape, strings
