#!/usr/bin/env python
"""PCIe H2D/D2H bandwidth from pinned memory: one stream vs split across
several streams (copy engines), for the e2e lane design."""
import json
import torch

N = 561 << 20
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
res = {}
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = N // ns
    for rep in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        res[f"h2d_{ns}streams"] = round(N / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
    # D2H concurrently with H2D (full duplex)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
s1.wait_event(e0); s2.wait_event(e0)
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
res["duplex_each_GBps"] = round(N / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
print(json.dumps(res))
