for v in "-DSEL_RW2=3 -DSEL_CW2=19" "-DSEL_RW2=4 -DSEL_CW2=18" "-DSEL_RW2=2 -DSEL_CW2=20"; do
  SEL_EXTRA_NVCC_FLAGS="$v" python -m paper_1806_08901_b200.build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"
  for o in "" "groups=2" "groups=4" "groups=12" "lag_t=1" "lag_t=3"; do
    echo "  opts: $o"; SEL_OPTS="$o" timeout 300 python scripts/measure_all.py c2 2>&1 | grep "C2" | head -1
  done
done
python -m paper_1806_08901_b200.build > /dev/null 2>&1
