timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "config3_recipe or config4_recipe or batch_exact_small or batch_kernel_tiny or config1 or config2_recipe or test_config5_recipe or full_config4 or multi_eb_vs_oracle or debug" 2>&1 | tail -3
timeout 300 python scripts/measure_all.py c1,c3,c4 2>&1 | grep "^| C"
echo "-- C1 range_warps=0"; SEL_OPTS="range_warps=0" timeout 300 python scripts/measure_all.py c1 2>&1 | grep "^| C"
timeout 250 python scripts/probe_multi.py c3,c4 2>&1 | grep "tile=1"
