#!/bin/bash
# Tile-configuration sweep (developer tool): rebuild libsel.so per variant, time C2 / C1.
IFS=";" read -ra VARS <<< "${SWEEP_VARIANTS:-default}"
for v in "${VARS[@]}"; do
  [ "$v" = default ] && v=""
  SEL_EXTRA_NVCC_FLAGS="$v" python -m paper_1806_08901_b200.build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== variant: ${v:-default}"
  timeout 300 python scripts/probe_groups.py 2>&1 | grep "G=0"
done
python -m paper_1806_08901_b200.build > /dev/null 2>&1
