"""Build a kernel-variant copy of libpgk.so for A/B timing on the GPU box.

    python tools/build_variant.py NAME DEF=VAL [DEF=VAL ...]
    -> paper_2410_01231_b200/variants/libpgk_NAME.so  (load with PGK_LIB_PATH)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2410_01231_b200 import build_ext  # noqa: E402

name, defs = sys.argv[1], tuple(sys.argv[2:])
out = build_ext.PKG / "variants" / f"libpgk_{name}.so"
out.parent.mkdir(exist_ok=True)
print(build_ext.build(out=out, defines=defs))
