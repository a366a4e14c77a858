#!/usr/bin/env python3
"""Decode a config with its irregular slices rebuilt by another construction (e.g. PEG):
FER, undetected frames, iterations and step time (tools/try_ensemble.py's runner).

  python tools/try_construction.py C2 peg [BATCHES]
"""
import dataclasses
import importlib.util
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from cvsr_inputs import configs  # noqa: E402

spec = importlib.util.spec_from_file_location("te", os.path.join(os.path.dirname(__file__), "try_ensemble.py"))
te = importlib.util.module_from_spec(spec)
spec.loader.exec_module(te)

base = configs.CONFIGS[sys.argv[1]]
constr = sys.argv[2]
batches = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = dataclasses.replace(base, slices=tuple(dataclasses.replace(s, construction=constr) if s.kind == "irregular" else s
                                             for s in base.slices))
te.run(base, f"{base.name} config-model")
for k in range(batches):
    te.run(cfg, f"{base.name} {constr}", first_frame=k * base.frames)
