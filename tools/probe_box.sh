#!/bin/bash
# One-shot description of the GPU box: host, topology, link probe.
mkdir -p gpurun_out
{
  echo "== lscpu"; lscpu | head -30
  echo "== free"; free -g
  echo "== nvidia-smi"; nvidia-smi
  echo "== topo"; nvidia-smi topo -m
  echo "== pcie"; nvidia-smi -q | grep -A 12 -i "PCI$\|GPU Link Info" | head -60
  echo "== numa"; ls /sys/devices/system/node/ ; cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c
  echo "== ulimit"; ulimit -l
} > gpurun_out/box_info.txt 2>&1
# the probes are built here from their sources (binaries are not committed)
for p in probe_link probe_gather; do
  [ -x tools/$p ] || /usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a \
      -o tools/$p tools/$p.cu || exit 1
done
./tools/probe_link 8 > gpurun_out/probe_link.jsonl 2> gpurun_out/probe_link.err
python - << 'PY' >> gpurun_out/box_info.txt 2>&1
import os; print("cpu_count", os.cpu_count())
PY
