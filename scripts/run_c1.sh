for v in "" "-DSEL_CW2=22 -DSEL_RW2=0"; do
  SEL_EXTRA_NVCC_FLAGS="$v" python -m paper_1806_08901_b200.build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"
  for o in "" "range_warps=0" "groups=37" "groups=74"; do
    echo "  opts: $o"; SEL_OPTS="$o" timeout 300 python scripts/measure_all.py c1 2>&1 | grep "^| C"
  done
done
python -m paper_1806_08901_b200.build > /dev/null 2>&1
