#!/bin/bash
# slab schedule: tests + timing (tools/exp_slab.py) incl. C3 and slab-length variants for C5
make -s > /dev/null 2>&1
bash tools/gpu_slab.sh ${1:-slab3} "slab or recompute or c3_parity or c4_parity or c5_shape or modes_agree or soft_boundary or extrinsic or edge_configuration or underflow or status_edge or alpha_beta or live or chunked or graph" C5:32 C4:512 C3:2048 C2:65536
