"""Build an EXPERIMENT variant of the library with extra -D flags (A/B measurements only; the
product library is paper_2408_11049_b200/libmagicdec_b200.so, built by build.py with the
defaults).  usage: python tools/build_variant.py OUT.so -DFLAG=1 ...   then MD_LIB=OUT.so python ..."""
import glob
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_11049_b200 import build as B  # noqa: E402

out, flags = sys.argv[1], sys.argv[2:]
srcs = sorted(glob.glob(os.path.join(B.HERE, "csrc", "*.cu")))
B._nvcc(srcs, os.path.abspath(out), extra=["-DMD_BUILD"] + flags, force=True)
print("built", out, flags)
