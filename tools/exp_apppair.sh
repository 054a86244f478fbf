#!/bin/bash
# Live-window APP of the register-heavy shapes (C3, C5): scalar core (default) vs pair core, G sweep.
OUT=gpurun_out/exp_apppair; mkdir -p $OUT
for v in 20 0; do
  touch paper_1802_08483_b200/csrc/*.cu
  make -s -j16 all EXTRA="-DBSIDMAP_SCALAR_APP_MN_MAX=$v" > $OUT/build_$v.log 2>&1 || { tail $OUT/build_$v.log; continue; }
  for cfg in C5:32 C3:2048; do
    C=${cfg%%:*}; F=${cfg#*:}
    for G in 2 4 8 12; do
      BSIDMAP_APP_G=$G python bench.py --config $C --frames $F --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${C}_$v_$G.json 2>/dev/null
      python -c "import json; d=json.load(open('$OUT/${C}_$v_$G.json')); print('$C scalar_app_max=$v G=$G', round(d['ms_per_step'],2), 'p2', round(d['phase_ms']['lattice_pass2'],2))"
    done
  done
done
touch paper_1802_08483_b200/csrc/*.cu; make -s -j16 all > /dev/null 2>&1
