#!/bin/bash
# Config 5: block-size sweep 128..4096 on Transformer-Big (1 GPU; bench.py under
# torchrun covers the multi-GPU points).  One JSON line per block size.
for b in 128 256 512 1024 2048 4096; do
  timeout 900 python bench.py --block-size $b --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1
done
