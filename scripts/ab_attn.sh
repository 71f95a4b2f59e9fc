#!/bin/bash
# A/B timing of the attention path for build/ab/A.so vs B.so (dev aid)
for r in 1 2; do for v in A B; do
  echo "$v $(VQKV_LIB=build/ab/$v.so timeout 200 python scripts/attn_bench.py 2>&1 | grep -E 'ms/layer|attend ' | tr '\n' ' ')"
done; done
