#!/bin/bash
# Profiles at head for C2-C5 (per-GPU batches), the exact-zero support statistics, the re-run of the
# folded-row test.   usage (under gpurun): bash tools/gpu_r02o.sh <tag>
TAG=${1:-r02o}
OUT=gpurun_out/$TAG; mkdir -p $OUT
make -s > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "two_folded" > $OUT/pytest_folded.log 2>&1; tail -2 $OUT/pytest_folded.log
timeout 600 python tools/support_stats.py > $OUT/support_stats.txt 2>&1; cat $OUT/support_stats.txt
for cf in "C2 65536" "C3 2048" "C4 512" "C5 32"; do set -- $cf; timeout 1200 bash tools/gpu_prof.sh $TAG $1 $2 > /dev/null 2>&1; head -c 300 $OUT/$1/bench.json; echo; done
