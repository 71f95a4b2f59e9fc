#!/bin/bash
# A/B timing of build/ab/A.so vs build/ab/B.so on one box (dev aid), interleaved
for r in 1 2 3; do for v in A B; do
  echo "$v $(VQKV_LIB=build/ab/$v.so timeout 200 python scripts/ab_encode.py ${1:-32} 2>&1 | tail -1)"
done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
