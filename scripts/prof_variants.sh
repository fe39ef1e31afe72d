# per-CTA cycle breakdown of k_batch (SEL_BATCH_PROF) for a set of compile-time variants
#   PROF_VARIANTS="-DX;-DY" PROF_CFGS="4 6;3 13" bash scripts/prof_variants.sh
IFS=";" read -ra VARS <<< "${PROF_VARIANTS:-}"
IFS=";" read -ra CFGS <<< "${PROF_CFGS:-4 6}"
for v in "${VARS[@]:-}"; do
  SEL_EXTRA_NVCC_FLAGS="-DSEL_BATCH_PROF=1 $v" python -m paper_1806_08901_b200.build > /dev/null 2>&1 || echo "build failed"
  echo "== $v"
  for c in "${CFGS[@]}"; do timeout 300 python scripts/probe_timing.py $c 2>&1 | grep -v "^field"; done
done
python -m paper_1806_08901_b200.build > /dev/null 2>&1
