# Turn gpurun_out/r2final_* (tools/measure_r2_final.sh) into profiles/ (run in the repo root, after the GPU call)
set -e
for c in c1 c2 c3 c4 c5 dist1 ref; do tail -n 1 gpurun_out/r2final_bench_$c.log > profiles/r2final_bench_$c.json; done
for spec in c1:10000000 c2:100000000 c3:200000000 c4:100000000 c5:500000000; do
  IFS=: read c n <<< "$spec"
  python tools/phase_traffic.py gpurun_out/r2final_traffic_$c.csv $n > profiles/r2_traffic_$c.json
done
cp gpurun_out/r2final_launches_c5.csv profiles/r2final_launches_c5.csv
python tools/launch_list.py gpurun_out/r2final_launches_c5.csv "# C5 bench --steps 1 --warmup 3 (round 2, final: one-pass level 0 and level 1)" > profiles/r2final_launches_c5.txt
{ echo "# ncu --set full, C5 (LogNormal(0,2) 5e8 f64, one sort via tools/profile_sort.py), round 2 final (one-pass level 0 + level 1)";
  echo "# command: tools/measure_r2_final.sh (ncu serialises kernels with cold caches: use shares, not absolute sums)";
  python tools/ncu_summary.py gpurun_out/r2final_c5_full.ncu-rep --stalls; } > profiles/r2final_ncu_full_summary.txt
tail -n 3 gpurun_out/r2final_gputest.log > profiles/r2final_gputest.txt
