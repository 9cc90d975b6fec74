# Round-2 final measurement set (GPU box): the GPU suite, bench lines for every
# config, the one-rank distributed path, the reference arm, per-config DRAM
# traffic per phase (ncu counters over one sort), the C5 launch list, and one
# ncu --set full capture of the C5 sort's partition / base-case kernels.
# Outputs in gpurun_out/ (r2final_*); tools/launch_list.py, phase_traffic.py and
# ncu_summary.py turn them into profiles/.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2final_gputest.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/r2final_bench_c5.log 2>&1
for c in c1 c2 c3 c4; do python bench.py --config $c --steps 10 --warmup 3 --cpu-runs 3 --e2e-steps 1 > gpurun_out/r2final_bench_$c.log 2>&1; done
python bench.py --dist --steps 5 --warmup 3 --no-cpu > gpurun_out/r2final_bench_dist1.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2final_bench_ref.log 2>&1
for spec in c1:uniform:10000000 c2:normal:100000000 c3:mixgauss:200000000 c4:rootdups:100000000 c5:lognormal2:500000000; do
  IFS=: read c d n <<< "$spec"
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r2final_traffic_$c.csv python tools/profile_sort.py $d $n 1 > gpurun_out/r2final_ncu_traffic_$c.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2final_launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/r2final_ncu_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:k_(direct|scatter|hist|base_reg)' -c 30 \
    -o gpurun_out/r2final_c5_full python tools/profile_sort.py lognormal2 500000000 1 > gpurun_out/r2final_ncu_full.log 2>&1
