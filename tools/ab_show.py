#!/usr/bin/env python3
"""Summarise tools/ab.sh results: tok/s, SM clock, tok/s per GHz."""
import json
import sys

tag = sys.argv[1]
for line in open(f"gpurun_out/{tag}_index.txt"):
    i, v = line.rstrip("\n").split(" ", 1)
    try:
        d = json.loads(open(f"gpurun_out/{tag}_{i}.json").read().strip().splitlines()[-1])
        mhz = d["clocks"]["sm_mhz"] or 0
        print(f"{v:45s} {d['value']:8.1f} tok/s  {mhz:6.0f} MHz  {d['value'] / mhz * 1000 if mhz else 0:6.1f} per GHz")
    except Exception as e:  # noqa: BLE001
        print(f"{v:45s} failed: {e}")
