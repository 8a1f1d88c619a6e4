"""One workload, one factorisation kernel variant, a few factorisations (ncu target)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1904_02401_b200 import _lib, workloads as W  # noqa: E402

name, variant = sys.argv[1], int(sys.argv[2])
lib = _lib.load()
lib.alefsi_dev_set_fact_variant.argtypes = [ctypes.c_int]
lib.alefsi_dev_set_fact_variant(variant)
prob, mg, b, _ = W.build_device_solver(W.CONFIGS[name])
for _ in range(2):
    mg.factorize()
torch.cuda.synchronize()
