"""Batched species block inverse probe: python scripts/blk_probe.py [ns] [N]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import json  # noqa: E402

import bench  # noqa: E402

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 11
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
print(json.dumps(bench.block_lu(6542.7, nss=(ns,), N=N, reps=1)))
