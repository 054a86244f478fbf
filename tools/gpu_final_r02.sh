#!/bin/bash
# Round-2 final evidence at one source digest: build + smoke, the gpu suite, bench lines (C2 default,
# C3/C4/C5 per-GPU batches, J1, C5 RECOMPUTE = slab), ncu captures of C2-C5, compute-sanitizer.
# usage (under gpurun): bash tools/gpu_final_r02.sh <tag>
TAG=${1:-r02z}; OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s > /dev/null 2>&1
nproc > $OUT/nproc.txt
python -c "from paper_1802_08483_b200._lib import source_digest; print(source_digest())" > $OUT/digest.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/build_smoke.log 2>&1; tail -1 $OUT/build_smoke.log
timeout 1500 python -m pytest tests -q -m gpu --durations=15 > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_C2.json 2> $OUT/bench_C2.err
for cf in "C3 2048" "C4 512" "C5 32" "J1 65536"; do set -- $cf
  timeout 900 python bench.py --config $1 --frames $2 > $OUT/bench_$1.json 2> $OUT/bench_$1.err; done
timeout 900 python bench.py --config C5 --frames 32 --mode recompute > $OUT/bench_C5_recompute.json 2> $OUT/bench_C5_recompute.err
for c in C2 C3 C4 C5 J1 C5_recompute; do python -c "
import json; d=json.load(open('$OUT/bench_$c.json')); r=d['roofline']
print('$c', round(d['value'],1), round(d['ms_per_step'],2), r.get('frac'), r.get('frac_executed'), d['e2e']['value'] if d.get('e2e') else None, d['clocks'])" 2>&1 | tail -1; done
for cf in "C2 65536" "C3 2048" "C4 512" "C5 32"; do set -- $cf; timeout 1200 bash tools/gpu_prof.sh $TAG $1 $2 > /dev/null 2>&1; done
# compute-sanitizer is closed on this pool (runs under it left GPUs needing a reset)
