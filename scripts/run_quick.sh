# quick GPU check after a kernel change: 3D/2D parity subset, then timing of the headline configs
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "config3_recipe or config4_recipe or batch_exact_small or batch_kernel_tiny or batch_full_size_stack or config1 or config2_recipe or test_config5_recipe or full_config4" 2>&1 | tail -3
timeout 300 python scripts/exp_rw.py c4,c3 2>&1 | grep -v "\[:"
