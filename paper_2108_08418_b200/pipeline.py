"""One sliced-reconciliation step (Bob + Alice) composed from the C ABI.

Argument marshalling and buffer ownership only: every step of the hot path
runs in libcvsr.so kernels.  torch provides device memory and the stream.
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import torch

from . import cvsr


class SRPipeline:
    """Device buffers + loaded codes for `frames` sub-blocks of n symbols.

    codes[j] is a host code object with (n, m_checks, row_ptr, col_idx) or
    None for a disclosed slice.  Bob: quantise y, syndromes of coded slices,
    packed bits of disclosed slices.  Alice: cvsr_reconcile.
    """

    def __init__(self, m: int, edges, codes: Sequence, order: Sequence[int], sigma_n: float, n: int, frames: int,
                 device: torch.device, max_iter: int = 100, msg_clamp: float = 40.0, stream=None,
                 schedule: str = "default"):
        self.m, self.n, self.frames, self.device = m, n, frames, device
        self.order = list(order)
        self.sigma_n = float(sigma_n)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        self.ctx = cvsr.cvsr_ctx_create(device.index or 0, self.stream)
        self.q = cvsr.make_quantiser(edges)
        self.opts = cvsr.decode_opts(max_iter, msg_clamp, schedule)  # BP schedule: cvsr_decode_opts.flags
        self.code_h: List[Optional[int]] = []
        self.code_E: List[int] = []
        for c in codes:
            if c is None:
                self.code_h.append(None)
                self.code_E.append(0)
            else:
                if c.n != n:
                    raise ValueError("code length != n")
                self.code_h.append(cvsr.cvsr_code_load(self.ctx, c.n, c.m_checks, c.row_ptr, c.col_idx))
                self.code_E.append(c.n_edges)
        W = lambda bits: (bits + 31) // 32  # noqa: E731
        kw = dict(device=device)
        self.label_bob = torch.empty((frames, n), dtype=torch.uint8, **kw)
        self.synd = [torch.empty((frames, W(c.m_checks) if c is not None else W(n)), dtype=torch.int32, **kw)
                     for c in codes]
        self.label_alice = torch.empty((frames, n), dtype=torch.uint8, **kw)
        self.frame_ok = torch.empty((frames,), dtype=torch.uint8, **kw)
        self.verified = torch.empty((frames,), dtype=torch.uint8, **kw)
        self.hash_alice = torch.empty((frames, cvsr.CVSR_HASH_KEYS), dtype=torch.int64, **kw)
        self.hash_bob = torch.empty((frames, cvsr.CVSR_HASH_KEYS), dtype=torch.int64, **kw)
        self.iters = torch.empty((frames, m), dtype=torch.int32, **kw)
        self.codes = list(codes)

    def bob(self, y: torch.Tensor) -> None:
        cvsr.cvsr_quantise(self.ctx, self.q, y, self.frames * self.n, self.label_bob)
        for j in range(self.m):
            if self.code_h[j] is None:
                cvsr.cvsr_slice_bits(self.ctx, self.label_bob, self.frames, self.n, j, self.synd[j])
            else:
                cvsr.cvsr_syndrome(self.ctx, self.code_h[j], self.label_bob, self.frames, j, self.synd[j])

    def alice(self, x: torch.Tensor, want_stats: bool = False) -> Optional[dict]:
        return cvsr.cvsr_reconcile(self.ctx, self.m, self.code_h, self.order, self.q, self.sigma_n, x, self.synd,
                                   self.frames, self.n, self.opts, self.label_alice, self.frame_ok, self.iters,
                                   want_stats=want_stats)

    def verify(self, keys) -> None:
        """PAPER.md:90 hash check: verified = frame_ok AND hash(Alice) == hash(Bob) under each of the
        cvsr.CVSR_HASH_KEYS independent keys (fresh per call)."""
        cvsr.cvsr_verify(self.ctx, self.label_alice, self.label_bob, self.frame_ok, self.frames, self.n, keys,
                         self.verified, self.hash_alice, self.hash_bob)

    def step(self, x: torch.Tensor, y: torch.Tensor, want_stats: bool = False,
             key=None) -> Optional[dict]:
        """Bob, Alice and (keys given: a sequence of cvsr.CVSR_HASH_KEYS ints) the hash verification
        of one batch."""
        self.bob(y)
        st = self.alice(x, want_stats)
        if key is not None:
            self.verify(key)
        return st

    def count_errors(self):
        return cvsr.cvsr_count_errors(self.ctx, self.label_alice, self.label_bob, self.frame_ok, self.frames, self.n)

    def launches(self) -> int:
        return cvsr.cvsr_ctx_launch_count(self.ctx)

    def close(self) -> None:
        if self.ctx:
            cvsr.cvsr_ctx_sync(self.ctx)
            for h in self.code_h:
                if h:
                    cvsr.cvsr_code_free(h)
            cvsr.cvsr_ctx_destroy(self.ctx)
            self.ctx = 0


class SplitPipeline:
    """k SRPipelines over disjoint frame ranges, each on its own stream and host thread.

    Frames are independent, so the k reconciles of a step may run concurrently;
    while one split is in the low-occupancy tail of a slice (few frames still
    iterating) the other's kernels fill the GPU.  Results are bit-identical to
    a single pipeline (per-frame computation does not depend on batching).
    """

    def __init__(self, k: int, m: int, edges, codes: Sequence, order: Sequence[int], sigma_n: float, n: int,
                 frames: int, device: torch.device, max_iter: int = 100, msg_clamp: float = 40.0,
                 schedule: str = "default"):
        import concurrent.futures as cf
        self.k = k
        self.frames, self.n, self.m = frames, n, m
        bounds = [frames * i // k for i in range(k + 1)]
        self.ranges = [(bounds[i], bounds[i + 1]) for i in range(k)]
        self.streams = [torch.cuda.Stream(device) for _ in range(k)]
        self.parts = [SRPipeline(m, edges, codes, order, sigma_n, n, b - a, device, max_iter, msg_clamp, stream=s,
                                 schedule=schedule)
                      for (a, b), s in zip(self.ranges, self.streams)]
        self.pool = cf.ThreadPoolExecutor(max_workers=k)
        self.device = device

    def step(self, x: torch.Tensor, y: torch.Tensor, want_stats: bool = False, key: Optional[int] = None):
        main = torch.cuda.current_stream(self.device)
        ev = main.record_event()
        for s in self.streams:
            s.wait_event(ev)

        def run(i):
            a, b = self.ranges[i]
            with torch.cuda.stream(self.streams[i]):
                return self.parts[i].step(x[a:b], y[a:b], want_stats, key)

        res = list(self.pool.map(run, range(self.k)))
        for s in self.streams:
            main.wait_stream(s)
        if not want_stats:
            return None
        out = {key: 0 for key in ("frames", "frames_ok", "bits_reconciled")}
        for key in ("attempted", "converged", "iters_sum", "edge_iters"):
            out[key] = [sum(r[key][j] for r in res) for j in range(self.m)]
        for r in res:
            for key in ("frames", "frames_ok", "bits_reconciled"):
                out[key] += r[key]
        out["alice_seconds"] = max(r["alice_seconds"] for r in res)
        return out

    def count_errors(self):
        tot = [0, 0, 0]
        for p in self.parts:
            c = p.count_errors()
            tot = [a + b for a, b in zip(tot, c)]
        return tuple(tot)

    @property
    def iters(self):
        return torch.cat([p.iters for p in self.parts])

    @property
    def label_alice(self):
        return torch.cat([p.label_alice for p in self.parts])

    @property
    def verified(self):
        return torch.cat([p.verified for p in self.parts])

    @property
    def frame_ok(self):
        return torch.cat([p.frame_ok for p in self.parts])

    def launches(self) -> int:
        return sum(p.launches() for p in self.parts)

    def close(self) -> None:
        for p in self.parts:
            p.close()
        self.pool.shutdown()
