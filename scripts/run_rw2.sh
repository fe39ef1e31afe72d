for v in "-DSEL_CW2=14 -DSEL_STAGES2=3" "-DSEL_CW2=14"; do
  SEL_EXTRA_NVCC_FLAGS="$v" python -m paper_1806_08901_b200.build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"
  timeout 300 python scripts/measure_all.py c1,c2 2>&1 | grep "^| C"
done
python -m paper_1806_08901_b200.build > /dev/null 2>&1
