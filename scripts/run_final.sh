# end-of-session check: full GPU suite, smoke, the two bench lines, throughput table
set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02e_gputest.log 2>&1; tail -2 gpurun_out/r02e_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.log 2>&1; tail -1 gpurun_out/r02e_smoke.log
python bench.py > gpurun_out/r02e_bench_c4.jsonl 2> gpurun_out/r02e_bench_c4.err
python bench.py --config 2 --no-cpu-baseline > gpurun_out/r02e_bench_c2.jsonl 2> gpurun_out/r02e_bench_c2.err
timeout 900 python scripts/measure_all.py > gpurun_out/r02e_throughput.md 2>&1
