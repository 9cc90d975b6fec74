# ncu --set full of the C5 sort's kernels (one sort; the sample-sort and gated
# kernels are captured too but take microseconds)
timeout 1500 ncu --set full --import-source on --clock-control none -k 'regex:k_(direct|scatter|hist|base_reg)' -c 30 -o gpurun_out/r2f_c5_full python tools/profile_sort.py lognormal2 500000000 1 > gpurun_out/r2f_ncu.log 2>&1
