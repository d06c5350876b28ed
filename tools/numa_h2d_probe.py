#!/usr/bin/env python
"""Pinned-memory H2D / D2H / duplex bandwidth with the process (and hence the
first touch of the pinned pages) bound to each NUMA node in turn — does the
host side of the e2e path need NUMA placement next to the GPU?
usage: tools/numa_h2d_probe.py [--device 0]"""
import argparse
import glob
import json
import os
import subprocess
import sys


def nodes():
    out = {}
    for d in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
        cpus = open(os.path.join(d, "cpulist")).read().strip()
        out[int(d.rsplit("node", 1)[1])] = cpus
    return out


def parse(cpulist):
    s = set()
    for part in cpulist.split(","):
        if "-" in part:
            a, b = part.split("-")
            s.update(range(int(a), int(b) + 1))
        elif part:
            s.add(int(part))
    return s


def gpu_numa(dev):
    import torch
    bus = torch.cuda.get_device_properties(dev).pci_bus_id if hasattr(
        torch.cuda.get_device_properties(dev), "pci_bus_id") else None
    try:
        q = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader",
                            "-i", str(dev)], capture_output=True, text=True).stdout.strip()
        bdf = q.lower().replace("00000000:", "0000:")
        return int(open(f"/sys/bus/pci/devices/{bdf}/numa_node").read()), bdf
    except Exception as e:  # noqa: BLE001
        return None, str(e)


def child(dev):
    import torch
    torch.cuda.set_device(dev)
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1); h2.fill_(1)  # first touch on this node
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("h2d", "d2h", "duplex"):
        best = 0.0
        for _ in range(4):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_event(e0); s2.wait_event(e0)
            if name in ("h2d", "duplex"):
                with torch.cuda.stream(s1):
                    d.copy_(h, non_blocking=True)
            if name in ("d2h", "duplex"):
                with torch.cuda.stream(s2):
                    h2.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            gbs = n / (e0.elapsed_time(e1) * 1e-3) / 1e9
            best = max(best, gbs)
        res[name + "_gbs_each_way" if name == "duplex" else name + "_gbs"] = round(best, 1)
    print(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.device)
        return
    gnode, bdf = gpu_numa(a.device)
    out = {"gpu": a.device, "gpu_numa_node": gnode, "bdf": bdf, "nodes": {}}
    for node, cpus in nodes().items():
        env = dict(os.environ)
        cmd = [sys.executable, os.path.abspath(__file__), "--child", "--device", str(a.device)]
        r = subprocess.run(cmd, capture_output=True, text=True, env=env,
                           preexec_fn=lambda c=parse(cpus): os.sched_setaffinity(0, c))
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        out["nodes"][node] = {"cpus": cpus, **(json.loads(line[-1]) if line else {"err": r.stderr[-300:]})}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
