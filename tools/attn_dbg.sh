#!/bin/bash
# Attention pipeline decomposition: time the tc attention hook with parts switched off
# (SDV2_ATTN_DBG bits: 1 softmax, 2 all MMAs, 4 K/V loads, 8 PV MMAs, 16 S MMAs).
for pu in 0 1; do
  for d in 0 1 2 3 5 7 9 17; do
    echo "PU=$pu DBG=$d"; SDV2_ATTN_PER_UNIT=$pu SDV2_ATTN_DBG=$d timeout 60 python tools/time_attn.py 2>&1 | cut -c1-60
  done
done
