# end-of-session capture for the 2D shape: C2 bench, launch list and one ncu --set full
set -x
python bench.py --config 2 --no-cpu-baseline > gpurun_out/r02e_bench_c2.jsonl 2> gpurun_out/r02e_bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02e_launches_c2_bench.csv python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-rd --no-alt > gpurun_out/r02e_ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_batch -s 3 -c 1 -f -o gpurun_out/r02e_k_batch_c2 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-rd --no-alt > gpurun_out/r02e_ncufull_c2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.log 2>&1; cat gpurun_out/r02e_smoke.log
