import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2108_08418_b200 import cvsr
ctx = cvsr.cvsr_ctx_create(0, torch.cuda.current_stream())
n_in = 1 << 25; n_out = n_in // 2
seed = np.random.default_rng(1).integers(0, 1 << 32, (n_in + n_out) // 32 + 1, dtype=np.uint64).astype(np.uint32)
plan = cvsr.cvsr_pa_plan_create(ctx, n_in, n_out, seed)
x = torch.randint(-2**31, 2**31 - 1, (2, n_in // 32), dtype=torch.int32, device='cuda')
y = torch.empty((2, n_out // 32), dtype=torch.int32, device='cuda')
cvsr.cvsr_pa_hash(ctx, plan, 2, x, y)
torch.cuda.synchronize()
