#!/usr/bin/env python3
"""Build a variant of libcvsr.so with extra preprocessor defines for A/B runs.

  python tools/build_variant.py NAME DEF=VAL ...   ->  build/variants/NAME.so
  CVSR_LIB=build/variants/NAME.so python bench.py ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_08418_b200 import _build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(_build.ROOT, "build", "variants")
os.makedirs(out_dir, exist_ok=True)
print(_build.build(out=os.path.join(out_dir, name + ".so"), defines=defs))
