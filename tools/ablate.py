"""Time variants of the c2 workload (e.g. fewer self blocks) with bench.py's own harness.

    python tools/ablate.py N=1           # c2_inner with one self block
    python tools/ablate.py k=8 heads=2   # any ModelConfig override
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

over = {}
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    over[k] = v if k == "merge_mode" else int(v)
bench.CONFIGS["ablate"] = dict(bench.CONFIGS["c2_inner"], **over)
sys.argv = ["bench.py", "--config", "ablate", "--steps", "10", "--warmup", "3"]
bench.main()
