#!/bin/bash
# alpha/beta overlap sub-batches: 1 (off) vs 2 vs 4, per config (device-resident inputs)
for AB in 1 2 4; do
  echo "=== BSIDMAP_AB_SUB=$AB"
  for c in "C2 65536" "C3 2048" "C4 512" "C5 32"; do
    BSIDMAP_AB_SUB=$AB python tools/quick_time.py $c 0 | grep -E "frames/s|phases" | tail -2
  done
done
