LSORT_TRACE=1 python tools/profile_sort.py lognormal2 500000000 2 > gpurun_out/s12_trace_c5.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:k_(direct|scatter|hist|base_reg)' -c 14 -o gpurun_out/s12_c5_full python tools/profile_sort.py lognormal2 500000000 1 > gpurun_out/s12_ncu_full.log 2>&1
