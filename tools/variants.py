"""Build tuning variants of libareal_b200.so (compile-time knobs) into build/variants/.

    python tools/variants.py NAME=-DFLAG=VAL[,-DFLAG2=VAL] ...
Each variant is selected with `tools/kbench.py --lib build/variants/libareal_b200_NAME.so`
(paper_2505_24298_b200._lib.use_library before the first load).."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_24298_b200 import build as B  # noqa: E402

out = os.path.join(ROOT, "build", "variants")
os.makedirs(out, exist_ok=True)
for spec in sys.argv[1:]:
    name, flags = spec.split("=", 1)
    path = os.path.join(out, f"libareal_b200_{name}.so")
    old = B.LIB_PATH
    B.LIB_PATH = path
    try:
        B.build(force=True, extra_flags=tuple(f for f in flags.split(",") if f))
    finally:
        B.LIB_PATH = old
    print(path)
