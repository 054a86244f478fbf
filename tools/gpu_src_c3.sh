#!/bin/bash
# source-level hot spots of the C3 scalar live APP
OUT=gpurun_out/${1:-src3}; mkdir -p $OUT
make -s > /dev/null 2>&1
k=k_app_live_x1
ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $OUT/$k \
    python bench.py --config C3 --frames 2048 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $OUT/$k.log 2>&1
python tools/src_hot.py $OUT/$k.ncu-rep $k 40 > $OUT/${k}_hot.txt 2>&1
python tools/src_ops.py $OUT/$k.ncu-rep $k MOV LDS ISETP BRA FFMA > $OUT/${k}_ops.txt 2>&1
rm -f $OUT/$k.ncu-rep
head -45 $OUT/${k}_hot.txt
