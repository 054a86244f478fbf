#!/bin/bash
# Live-window APP variants: prefix-sharing length KP and folded rows KS per config (env overrides).
OUT=gpurun_out/exp_kpks; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for cfg in C2 C5:32 C3:2048 C4:512; do
  C=${cfg%%:*}; F=${cfg#*:}; [ "$F" = "$cfg" ] && F=""
  for kp in 0 2 3 4; do for ks in 1 2; do
    BSIDMAP_APP_KP=$kp BSIDMAP_APP_KS=$ks python bench.py --config $C ${F:+--frames $F} --steps 4 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/${C}_$kp$ks.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/${C}_$kp$ks.json')); print('$C KP=$kp KS=$ks', round(d['ms_per_step'],2), 'p2', round(d['phase_ms']['lattice_pass2'],2))" 2>/dev/null || echo "$C KP=$kp KS=$ks failed"
  done; done
done
