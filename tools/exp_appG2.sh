#!/bin/bash
OUT=gpurun_out/exp_appG2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for cfg in C2 C5:32 C3:2048 C4:512; do
  C=${cfg%%:*}; F=${cfg#*:}; [ "$F" = "$cfg" ] && F=""
  for G in auto 4 8 12; do
    if [ $G = auto ]; then unset BSIDMAP_APP_G; else export BSIDMAP_APP_G=$G; fi
    python bench.py --config $C ${F:+--frames $F} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${C}_G$G.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/${C}_G$G.json')); print('$C G=$G', d['config']['app_frames_per_warp'], round(d['config']['live_windows_per_row'] or 0,2), round(d['ms_per_step'],2), 'p2', round(d['phase_ms']['lattice_pass2'],2), 'ab', round(d['phase_ms']['alpha_beta_busy'],2))"
  done
done
unset BSIDMAP_APP_G
timeout 600 python -m pytest tests -q -m gpu -k "graph or wide_trellis or packing" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
