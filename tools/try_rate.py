#!/usr/bin/env python3
"""C2 with a different rate / lambda for one slice: FER, undetected frames, iterations, step time.

  python tools/try_rate.py SLICE RATE 'LAMBDA_JSON' [BATCHES]
"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from cvsr_inputs import configs  # noqa: E402
import importlib.util  # noqa: E402

spec = importlib.util.spec_from_file_location("te", os.path.join(os.path.dirname(__file__), "try_ensemble.py"))
te = importlib.util.module_from_spec(spec)
spec.loader.exec_module(te)

j, rate = int(sys.argv[1]), float(sys.argv[2])
lam = json.loads(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] else None
batches = int(sys.argv[4]) if len(sys.argv) > 4 else 2
base = configs.C2
slices = tuple(dataclasses.replace(s, rate=rate, lam=tuple(sorted((int(a), float(w)) for a, w in lam.items())) if lam else s.lam)
               if s.j == j else s for s in base.slices)
cfg = dataclasses.replace(base, slices=slices)
for k in range(batches):
    te.run(cfg, f"C2 S{j} R={rate}", first_frame=k * base.frames)
