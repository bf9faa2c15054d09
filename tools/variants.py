"""Build tuning variants of libvlr.so (extra -D defines) under tools/_variants/
(git-ignored, travels to the GPU box) -- timing experiments only.

python tools/variants.py NAME DEF=VAL [DEF=VAL ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_08930_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_variants", name, "libvlr.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(b.build(out=out, defines=defs))
