"""Does a kernel on stream B run while isc_debug_occupy holds part of the GPU
on stream A?  Prints the wall time until B's work completes."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1611_09048_b200 import _abi  # noqa: E402

lib = _abi.lib()
import os
MODE = os.environ.get('MODE', 'add')
a, b = torch.cuda.Stream(), torch.cuda.Stream()
x = torch.zeros(1 << 20, device="cuda")
torch.cuda.synchronize()
cfgs = [tuple(int(v) for v in c.split('x')) for c in sys.argv[1:]] or [(148, 1024), (64, 128), (1, 32)]
for ctas, threads in cfgs:
    t0 = time.perf_counter()
    _abi.check(lib.isc_debug_occupy(ctas, threads, int(1e9), a.cuda_stream), "occupy")
    time.sleep(0.05)
    with torch.cuda.stream(b):
        if MODE == "add":
            x.add_(1)
        else:
            y = x.sum()     # block reduction: needs shared memory
    ev = torch.cuda.Event()
    ev.record(b)
    while not ev.query():
        pass
    t_b = time.perf_counter() - t0
    torch.cuda.synchronize()
    print(f"hog {ctas}x{threads}: stream-B kernel done after {t_b:.3f}s, hog done after {time.perf_counter() - t0:.3f}s",
          flush=True)
