#!/bin/bash
# Compile-time variant sweep (developer tool): rebuild libsel.so per variant and run
# measure_all.py on the selected configs.
#   SWEEP_VARIANTS="default;-DSEL_RWARPS=2" SWEEP_CFGS=c2,c3 bash scripts/sweep.sh
IFS=";" read -ra VARS <<< "${SWEEP_VARIANTS:-default}"
for v in "${VARS[@]}"; do
  [ "$v" = default ] && v=""
  SEL_EXTRA_NVCC_FLAGS="$v" python -m paper_1806_08901_b200.build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== variant: ${v:-default}"
  timeout 600 python scripts/measure_all.py "${SWEEP_CFGS:-c2,c3}" 2>&1 | grep "^| C"
done
python -m paper_1806_08901_b200.build > /dev/null 2>&1
