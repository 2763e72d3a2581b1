#!/usr/bin/env python
"""Build A/B variants of libtamp.so with extra -D defines (and nvcc flags after '|') into exp/<name>/ (git-ignored,
travels to the GPU box).
    python tools/build_variants.py name:DEF=1,DEF2=0 name2:DEF=2 "name3:|-Xptxas|--allow-expensive-optimizations=true" ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_11833_b200 import build as b  # noqa: E402

for arg in sys.argv[1:]:
    name, _, rest = arg.partition(":")
    defs, _, flags = rest.partition("|")
    print(name, b.build_variant(name, [d for d in defs.split(",") if d], flags=[f for f in flags.split("|") if f]),
          flush=True)
