set -x
python -m pytest tests -m gpu -x -q > gpurun_out/s4f_gputest.log 2>&1; tail -3 gpurun_out/s4f_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4f_smoke.log 2>&1; tail -2 gpurun_out/s4f_smoke.log
python bench.py > gpurun_out/s4f_bench.json 2> gpurun_out/s4f_bench.err; tail -c 600 gpurun_out/s4f_bench.json
python bench.py --impl reference > gpurun_out/s4f_bench_reference.json 2> gpurun_out/s4f_bench_reference.err; tail -c 400 gpurun_out/s4f_bench_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s4f_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-ttt --no-cpu-baseline --no-small > gpurun_out/s4f_ncu.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_ix_product -s 8 -c 2 --csv --log-file gpurun_out/s4f_traffic.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-ttt --no-cpu-baseline --no-small > gpurun_out/s4f_ncu2.log 2>&1
python tools/level_steps.py > gpurun_out/s4f_levels.log 2>&1
python tools/small_phases.py > gpurun_out/s4f_small.log 2>&1
