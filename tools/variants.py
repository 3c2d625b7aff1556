"""Build tuning variants of libvplgi.so (tools/ only): python tools/variants.py NAME DEF=V ..."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2203_11484_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], tuple(sys.argv[2:])
print(B.build(defines=defs, out=B.PKG / f"libvplgi_{name}.so"))
