# Round-2 measurement set (GPU box): bench lines for every config, the
# reference arm on the default config, per-config DRAM traffic per phase
# (ncu counters over one sort), the C5 launch list, and an ncu --set full
# capture of the top kernels. Outputs in gpurun_out/.
set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/r2m_bench_c5.log 2>&1
for c in c1 c2 c3 c4; do python bench.py --config $c --steps 10 --warmup 3 --cpu-runs 3 --e2e-steps 1 > gpurun_out/r2m_bench_$c.log 2>&1; done
python bench.py --dist --steps 5 --warmup 3 > gpurun_out/r2m_bench_dist1.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2m_bench_ref.log 2>&1
for spec in c1:uniform:10000000 c2:normal:100000000 c3:mixgauss:200000000 c4:rootdups:100000000 c5:lognormal2:500000000; do
  IFS=: read c d n <<< "$spec"
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r2m_traffic_$c.csv python tools/profile_sort.py $d $n 1 > gpurun_out/r2m_ncu_traffic_$c.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m_launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/r2m_ncu_launch.log 2>&1
