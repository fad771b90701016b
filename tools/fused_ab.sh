#!/bin/bash
# A/B of the fused IN+MID wide unit: config-4 stages and 64 config-2 frames for each
# library given (default build first), plus the unfused three-launch reference.
cd "$(dirname "$0")/.."
for lib in paper_1801_02108_b200/libsbnet.so "$@"; do
  SBN_LIB_PATH=$lib timeout 200 python tools/backbone_stages.py 8 0.2 2>&1 | grep -v Warn
  SBN_LIB_PATH=$lib timeout 120 python tools/wide_ab.py "$lib" 2>&1 | grep -v Warn
done
SBN_FLAGS=256 timeout 200 python tools/backbone_stages.py 8 0.2 2>&1 | grep -v Warn
SBN_FLAGS=256 timeout 120 python tools/wide_ab.py unfused 2>&1 | grep -v Warn
