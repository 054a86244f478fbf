#!/bin/bash
# Live-window APP: frames per warp G (partly filled rounds vs per-frame smem sums).
OUT=gpurun_out/exp_appG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for cfg in C2 C5:32 C3:2048; do
  C=${cfg%%:*}; F=${cfg#*:}; [ "$F" = "$cfg" ] && F=""
  for G in 4 8 12 16; do
    BSIDMAP_APP_G=$G python bench.py --config $C ${F:+--frames $F} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${C}_G$G.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/${C}_G$G.json')); print('$C G=$G', round(d['ms_per_step'],2), 'pass2', round(d['phase_ms']['lattice_pass2'],2))"
  done
done
