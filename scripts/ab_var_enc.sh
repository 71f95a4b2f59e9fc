#!/bin/bash
# A/B timing of build/var/<name>.so encoder variants (dev aid), interleaved
for r in 1 2 3; do for v in "$@"; do
  echo "$v $(VQKV_LIB=build/var/$v.so timeout 200 python scripts/ab_encode.py 32 2>&1 | tail -1)"
done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
