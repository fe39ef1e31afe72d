# end-of-session capture: default bench (C4), C2 bench, launch lists and one ncu --set full each
set -x
python bench.py > gpurun_out/r02e_bench_c4.jsonl 2> gpurun_out/r02e_bench_c4.err
python bench.py --config 2 --no-cpu-baseline > gpurun_out/r02e_bench_c2.jsonl 2> gpurun_out/r02e_bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02e_launches_c4_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-rd --no-alt > gpurun_out/r02e_ncu_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02e_launches_c2_bench.csv python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-rd --no-alt > gpurun_out/r02e_ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_batch -s 3 -c 1 -o gpurun_out/r02e_k_batch_c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-rd --no-alt > gpurun_out/r02e_ncufull_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_batch -s 3 -c 1 -o gpurun_out/r02e_k_batch_c2 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-rd --no-alt > gpurun_out/r02e_ncufull_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tile_multi -s 1 -c 1 -o gpurun_out/r02e_k_tile_multi_c3 python scripts/probe_multi.py c3 > gpurun_out/r02e_ncufull_multi.log 2>&1
ls -la gpurun_out | tail -20
