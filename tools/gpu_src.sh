#!/bin/bash
# source-level hot spots of the C2 lattice kernels (ncu --import-source, report kept on the box only)
OUT=gpurun_out/${1:-src}; mkdir -p $OUT
make -s > /dev/null 2>&1
for k in k_app_live k_gamma_sum; do
  ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $OUT/$k \
      python bench.py --config C2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $OUT/$k.log 2>&1
  python tools/src_hot.py $OUT/$k.ncu-rep $k 40 > $OUT/${k}_hot.txt 2>&1
  python tools/src_ops.py $OUT/$k.ncu-rep $k > $OUT/${k}_ops.txt 2>&1
  rm -f $OUT/$k.ncu-rep
done
head -60 $OUT/k_app_live_ops.txt
