SEL_EXTRA_NVCC_FLAGS="-DSEL_BATCH_PROF=1" python -m paper_1806_08901_b200.build > /dev/null 2>&1 || echo "build failed"
timeout 300 python scripts/prof_data.py 2>&1
timeout 300 python scripts/prof_rw.py 2 36 2>&1
timeout 300 python scripts/prof_rw.py 4 6 2>&1
python -m paper_1806_08901_b200.build > /dev/null 2>&1
