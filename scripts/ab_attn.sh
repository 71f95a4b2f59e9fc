#!/bin/bash
# A/B timing of build/ab/A.so vs build/ab/B.so for decode attention (dev aid), interleaved
for r in 1 2; do for v in A B; do
  echo "$v $(VQKV_LIB=build/ab/$v.so timeout 200 python scripts/attn_bench.py --gm 2>&1 | grep -E 'layer-step|ms/launch' | sed -E 's/attention ctx=[0-9]+ pairs=[0-9]+: //; s/ +/ /g' | tr '\n' ' ')"
done; done
