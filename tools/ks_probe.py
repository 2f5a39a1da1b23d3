"""Key-switch rates (bench.keyswitch_rate) at the bench shape, without the
rest of the bench.   python tools/ks_probe.py [lvl] [bsz]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_09164_b200.ckks.engine import CkksBackend
from paper_2104_09164_b200.ckks.params import gen_params
import bench
lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 12
bsz = int(sys.argv[2]) if len(sys.argv) > 2 else 64
be = CkksBackend(gen_params("fast-hear"), seed=0)
print(os.environ.get("TAG", ""), bench.keyswitch_rate(be, lvl, bsz), flush=True)
