"""Pinned host -> device copy rate with 1, 2 and 4 concurrent streams (is one
copy engine or the PCIe link the e2e ceiling?).  python tools/h2d_probe.py"""
import json

import torch

dev = torch.device("cuda", 0)
n = 4 << 30
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
host.fill_(1)
dbuf = torch.empty(n, dtype=torch.uint8, device=dev)
out = {}
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream(dev) for _ in range(ns)]
    part = n // ns
    best = 0.0
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                dbuf[i * part:(i + 1) * part].copy_(host[i * part:(i + 1) * part], non_blocking=True)
        for s in streams:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else torch.cuda.current_stream().wait_stream(s)
        torch.cuda.current_stream().wait_stream(streams[-1])
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    out[f"{ns}_streams_GBps"] = round(best, 2)
# device -> host for reference
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
host.copy_(dbuf, non_blocking=True)
e1.record()
torch.cuda.synchronize()
out["d2h_GBps"] = round(n / (e0.elapsed_time(e1) / 1e3) / 1e9, 2)
print(json.dumps(out))
