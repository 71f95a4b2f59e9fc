#!/bin/bash
# A/B timing of build/var/<name>.so variants for decode attention (dev aid), interleaved
for r in $(seq ${AB_ROUNDS:-3}); do for v in "$@"; do
  echo "$v $(VQKV_LIB=build/var/$v.so timeout 200 python scripts/attn_bench.py --gm 2>&1 | grep -E 'layer-step|ms/launch' | sed -E 's/attention ctx=[0-9]+ pairs=[0-9]+: //; s/ +/ /g' | tr '\n' ' ')"
done; done
