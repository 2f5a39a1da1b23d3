"""Run the key-switch ModUp NTT launch a few times (ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_09164_b200.ckks.engine import CkksBackend
from paper_2104_09164_b200.ckks.params import gen_params
import bench
be = CkksBackend(gen_params("fast-hear"), seed=0)
print(bench.dominant_kernel_roofline(be, lvl=6, bsz=16, peaks={}))
