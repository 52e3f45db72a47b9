"""Build liblofp_<name>.so with extra nvcc defines (A/B experiments; load with LOFP_LIB)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_26408_b200 import _build as b

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.HERE, f"liblofp_{name}.so")
subprocess.check_call([b.nvcc()] + b.NVCC_FLAGS + [f"-D{d}" for d in defs] + ["-o", out] + b.SOURCES)
print(out)
