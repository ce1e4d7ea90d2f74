"""One config-5 launch (for ncu): python tools/c5_one.py M R D LAYOUT"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_06619_b200 import _ext  # noqa: E402

m, r, d, lay = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), sys.argv[4]
print(_ext.bench_maxplus(m, m, r, d, seed=7, reps=2, flush_l2=True, layout=lay))
