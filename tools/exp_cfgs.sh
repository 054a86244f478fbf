#!/bin/bash
# timing of every config (subset batches) through quick_time
make -j16 >/dev/null 2>&1
python tools/quick_time.py C1 16384 0 | grep -E "TF/s|phases" | tail -2
python tools/quick_time.py C3 1024 0 | grep -E "TF/s|phases" | tail -2
python tools/quick_time.py C4 256 0 | grep -E "TF/s|phases" | tail -2
python tools/quick_time.py C5 32 0 | grep -E "TF/s|phases" | tail -2
