"""Run bench.py with cudaLimitMaxL2FetchGranularity set first (tuning experiment for the cfg5
partial-line over-fetch): python tools/l2fetch_run.py <bytes> <bench args...>"""
import ctypes
import os
import runpy
import sys

import torch

gran = int(sys.argv[1])
torch.cuda.init()
torch.zeros(1, device="cuda")                 # primary context
rt = ctypes.CDLL("libcudart.so.12")
cudaLimitMaxL2FetchGranularity = 0x05
rc = rt.cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, ctypes.c_size_t(gran))
v = ctypes.c_size_t(0)
rt.cudaDeviceGetLimit(ctypes.byref(v), cudaLimitMaxL2FetchGranularity)
print("l2 fetch granularity: set rc=%d, now %d" % (rc, v.value), file=sys.stderr)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
sys.argv = [os.path.join(root, "bench.py")] + sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
