"""GPU child of test_layered_decode_parity: decodes the cases in argv[1] (npz) through the C ABI
with the schedule the parent put in CVSR_SCHEDULE and writes bits / converged / iters to argv[2].
Imports only the CUDA binding (no oracle)."""
import sys

import numpy as np
import torch

from paper_2108_08418_b200 import cvsr as cv


def main():
    src = np.load(sys.argv[1])
    out = {}
    ctx = cv.cvsr_ctx_create(0, torch.cuda.current_stream())
    for name in src["names"]:
        n, M, max_iter = (int(v) for v in src[f"{name}_dims"])
        rp, ci = src[f"{name}_rp"], src[f"{name}_ci"]
        llr, synd = src[f"{name}_llr"], src[f"{name}_synd"]
        F = llr.shape[0]
        h = cv.cvsr_code_load(ctx, n, M, rp, ci)
        bits = torch.empty((F, (n + 31) // 32), dtype=torch.int32, device="cuda")
        conv = torch.empty(F, dtype=torch.uint8, device="cuda")
        iters = torch.empty(F, dtype=torch.int32, device="cuda")
        cv.cvsr_decode(ctx, h, torch.from_numpy(llr).cuda(), torch.from_numpy(synd.view(np.int32)).cuda(), F,
                       cv.decode_opts(max_iter, 40.0), bits, conv, iters)
        cv.cvsr_ctx_sync(ctx)
        cv.cvsr_code_free(h)
        out[f"{name}_bits"] = bits.cpu().numpy().view(np.uint32)
        out[f"{name}_conv"] = conv.cpu().numpy()
        out[f"{name}_iters"] = iters.cpu().numpy()
    cv.cvsr_ctx_destroy(ctx)
    np.savez(sys.argv[2], **out)


if __name__ == "__main__":
    main()
