"""Scratch: run R concurrent binary_swap ranks on one GPU and dump flag blocks."""
import sys, threading, ctypes as C, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1611_09048_b200 as P

R = int(sys.argv[1]); epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
h, w = 37, 29
grp = P.LocalNvlinkGroup(R, h * w)
order = list(np.random.default_rng(R).permutation(R))
imgs = [torch.rand((h, w, 4), device="cuda") for _ in range(R)]
errs = []
log = []
def body(r):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ep = grp.endpoints[r]; ep.n_ctas = 2; ep.timeout_s = 3.0
        for e in range(epochs):
            try:
                P.binary_swap(ep, imgs[r], order)
                log.append((r, e, "ok"))
            except Exception as exc:
                errs.append((r, e, str(exc)[:60])); return
ts = [threading.Thread(target=body, args=(r,)) for r in range(R)]
[t.start() for t in ts]; [t.join(60) for t in ts]
torch.cuda.synchronize()
print("errors", errs)
print("log", sorted(log))
for r, a in enumerate(grp.arenas):
    f = (C.c_ulonglong * 16)()
    torch.cuda.synchronize()
    C.memmove(f, 0, 0)
    t = a.tensor(a.flags_ptr, (32,)).view(torch.int64).cpu().tolist()
    print("rank", r, "flags", t[:10])
