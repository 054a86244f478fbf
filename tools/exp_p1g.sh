#!/bin/bash
# Pass 1 of the register-heavy pair shapes (C3, C4, C5, J1): row pairs (BSIDMAP_L1_GROUP) x CTAs/SM
# of the class kernel (BSIDMAP_L1C_MINB_LOW); compile-time knobs, one build each.
OUT=gpurun_out/exp_p1g; mkdir -p $OUT
for v in "1 3" "2 3" "2 2" "1 2"; do
  set -- $v; G=$1; M=$2
  make -s -j16 all EXTRA="-DBSIDMAP_L1_GROUP=$G -DBSIDMAP_L1C_MINB_LOW=$M" > $OUT/build_$G$M.log 2>&1 || { tail $OUT/build_$G$M.log; continue; }
  for cfg in C5:32 C3:2048 J1; do
    C=${cfg%%:*}; F=${cfg#*:}; [ "$F" = "$cfg" ] && F=""
    python bench.py --config $C ${F:+--frames $F} --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/${C}_$G$M.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/${C}_$G$M.json')); print('$C group=$G minb=$M', round(d['ms_per_step'],2), 'p1', round(d['phase_ms']['lattice_pass1'],2))"
  done
  touch paper_1802_08483_b200/csrc/*.cu
done
