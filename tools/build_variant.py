"""Build a tuning variant of libadimaxwell.so under build/variants/<name>/ (sweep tiling via -D).

    python tools/build_variant.py NAME CH_MASS RS_MASS CH_MOD RS_MOD CH_DER RS_DER
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_06998_b200 as adi  # noqa: E402

name, *v = sys.argv[1:]
keys = ["CH_MASS", "RS_MASS", "CH_MOD", "RS_MOD", "CH_DER", "RS_DER", "MINB_MASS"]
flags = ["-DADI_SW_TUNE"] + [f"-DADI_SW_{k}={x}" for k, x in zip(keys, v)]
path = os.path.join(ROOT, "build", "variants", name, "libadimaxwell.so")
print(adi.build(force=True, lib_path=path, extra_flags=flags))
