#!/bin/bash
# branch-free ceiling of the APP pass: a compile-time codeword (results invalid; timing only)
for V in "" "-DBSIDMAP_FAKE_X=0x2a5u"; do
  make clean >/dev/null; make -j$(nproc) EXTRA="$V" >/dev/null 2>&1 || { echo "build failed: $V"; continue; }
  BSIDMAP_APP_KP=0 KTAG="[$V KP=0]" python tools/ktime.py C2:65536
done
make clean >/dev/null; make -j$(nproc) >/dev/null 2>&1
