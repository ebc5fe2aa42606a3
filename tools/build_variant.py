"""Build a tuning variant of libadimaxwell.so under build/variants/<name>/ with extra -D flags.

    python tools/build_variant.py NAME [--degrees 2] -DADI_ST_WARPS_MASS=8 ...

Only the listed degrees are compiled (the others are stubs); select the build with ADI_LIB=<path>.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2103_06998_b200 as adi  # noqa: E402

args = sys.argv[1:]
name = args.pop(0)
degrees = adi.DEGREES
if args and args[0] == "--degrees":
    args.pop(0)
    degrees = tuple(int(x) for x in args.pop(0).split(","))
path = os.path.join(ROOT, "build", "variants", name, "libadimaxwell.so")
print(adi.build(force=True, lib_path=path, extra_flags=args, degrees=degrees))
