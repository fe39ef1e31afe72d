for v in "-DSEL_RW2=1" "-DSEL_W3=10240"; do
  SEL_EXTRA_NVCC_FLAGS="$v" python -m paper_1806_08901_b200.build > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "== $v"
  timeout 300 python scripts/measure_all.py c2,c3,c4 2>&1 | grep "^| C" | grep -v "N1\|(4, 4"
done
python -m paper_1806_08901_b200.build > /dev/null 2>&1
