# Round measurement set (GPU box): bench lines for every config, the C2 launch
# list and the per-phase DRAM traffic of one C2 sort. Outputs in gpurun_out/.
set -x
python bench.py > gpurun_out/bench_c2.log 2>&1
for c in c1 c3 c4 c5; do python bench.py --config $c --no-cpu --e2e-steps 1 > gpurun_out/bench_$c.log 2>&1; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/traffic_normal.csv python tools/profile_sort.py normal 100000000 1 > gpurun_out/ncu_traffic.log 2>&1
python bench.py --dist --no-cpu --e2e-steps 2 > gpurun_out/bench_dist1.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_all.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
