# end-of-session check: full GPU suite, smoke, the two bench lines, launch list + ncu --set full of the C4 bench, throughput table
set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02e_gputest.log 2>&1; tail -2 gpurun_out/r02e_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.log 2>&1; tail -1 gpurun_out/r02e_smoke.log
python bench.py > gpurun_out/r02e_bench_c4.jsonl 2> gpurun_out/r02e_bench_c4.err
python bench.py --config 2 --no-cpu-baseline > gpurun_out/r02e_bench_c2.jsonl 2> gpurun_out/r02e_bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02e_launches_c4_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-rd --no-alt > gpurun_out/r02e_ncu_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_batch -s 3 -c 1 -f -o gpurun_out/r02e_k_batch_c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-rd --no-alt > gpurun_out/r02e_ncufull_c4.log 2>&1
timeout 900 python scripts/measure_all.py > gpurun_out/r02e_throughput.md 2>&1
