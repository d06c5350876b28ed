#!/usr/bin/env python
"""Re-fit the b200 cost-model profile (north_star: "the
runtime tuner, re-fit to measured B200 HBM and NVLink latency and
bandwidth") from the K5 probes of THIS box, and write every value's source.

  local : dependent-load latency (1 GiB random cycle) and random-row gather
          bandwidth -> localLoadBase, perElemLocal
  peer  : (only when >= 2 GPUs are visible) the same from device 0 into
          device 1's HBM over NVLink -> remoteGetBase, perElemRemote
          (with one GPU these keep their previous value and source)

usage: tools/refit_b200.py [--write] [--out gpurun_out/refit.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PROFILE = os.path.join(ROOT, "paper_2209_06800_b200", "profiles", "b200.json")


def measure():
    from paper_2209_06800_b200 import probes
    m = {"local_chase_ns": probes.chase_ns(1 << 30),
         "local_gather_gbps": probes.gather_gbps(2_449_029, 16, 60_000_000),
         "devices": probes.device_count()}
    if m["devices"] >= 2:
        m["peer_chase_ns"] = probes.peer_chase_ns(0, 1)
        m["peer_gather_gbps"] = probes.peer_gather_gbps(0, 1, 2_449_029, 16, 30_000_000)
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--write", action="store_true", help="rewrite the b200 profile")
    ap.add_argument("--out", default=None)
    ap.add_argument("--sm-ghz", type=float, default=1.965)
    args = ap.parse_args()
    from paper_2209_06800_b200 import probes
    prof = json.load(open(PROFILE))
    m = measure()
    fit = probes.refit_latencies(m, args.sm_ghz, prof["numSMs"])
    prof["latencies"].update(fit["latencies"])
    prof["source"].update(fit["source"])
    rec = {"measured": m, "profile": prof}
    print(json.dumps(rec, indent=1))
    if args.out:
        json.dump(rec, open(args.out, "w"), indent=1)
    if args.write:
        json.dump(prof, open(PROFILE, "w"), indent=2)
        open(PROFILE, "a").write("\n")


if __name__ == "__main__":
    main()
