#!/usr/bin/env python3
"""Toeplitz privacy amplification throughput on one B200.

PA input: the reconciled bit string cut into blocks of n_in bits, each hashed to
n_out = ratio * n_in bits with the plan's seed.  Prints one JSON line per size:
input bits/s, the per-block time, and the DRAM-traffic roofline of the NTT passes.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_08418_b200 import cvsr  # noqa: E402


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6453.1}
    stream = torch.cuda.current_stream()
    ctx = cvsr.cvsr_ctx_create(0, stream)
    rng = np.random.default_rng(5)
    for lg_in, ratio, blocks in ((20, 0.5, 64), (23, 0.5, 16), (25, 0.5, 8), (26, 0.9, 4)):
        n_in = 1 << lg_in
        n_out = int(n_in * ratio)
        seed = rng.integers(0, 1 << 32, (n_in + n_out - 1 + 31) // 32, dtype=np.uint64).astype(np.uint32)
        plan = cvsr.cvsr_pa_plan_create(ctx, n_in, n_out, seed)
        N = cvsr.cvsr_pa_plan_info(plan)[2]
        x = torch.randint(-2 ** 31, 2 ** 31 - 1, (blocks, n_in // 32), dtype=torch.int32, device="cuda")
        y = torch.empty((blocks, (n_out + 31) // 32), dtype=torch.int32, device="cuda")
        for _ in range(2):
            cvsr.cvsr_pa_hash(ctx, plan, blocks, x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 5
        e0.record(stream)
        for _ in range(K):
            cvsr.cvsr_pa_hash(ctx, plan, blocks, x, y)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K / blocks
        lg = N.bit_length() - 1
        P = -(-max(lg - 12, 0) // 4)  # global radix-16 passes per direction
        # design bytes: first DIF pass reads the packed bits and writes N words; the other 2P - 1
        # global passes read + write N words; the shared-memory kernel reads data + seed transform
        # and writes data; the pack reads the n_out-word window and writes n_out bits
        traffic = n_in / 8 + 4 * N + (2 * P - 1) * 8 * N + 12 * N + 4 * n_out + n_out / 8
        print(json.dumps({"workload": "toeplitz_pa", "n_in": n_in, "n_out": n_out, "ntt_size": N, "blocks": blocks,
                          "ms_per_block": ms, "input_bits_per_s": n_in / (ms * 1e-3),
                          "output_bits_per_s": n_out / (ms * 1e-3),
                          "roofline": {"bound": "hbm", "achieved": traffic / (ms * 1e-3) / 1e9,
                                       "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                       "frac": traffic / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                       "note": "design bytes of the transform passes (not ncu)"}}), flush=True)
        cvsr.cvsr_pa_plan_free(plan)
    cvsr.cvsr_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
