python tools/ab_total.py --dists lognormal2:5e8,normal:1e8,mixgauss:2e8,uniform:1e7 --reps 4 --variants "bucket_target=4096;bucket_target=2048;bucket_target=8192;rmi_sample_cap=262144;rmi_sample_cap=524288" > gpurun_out/s3_ab.log 2>&1
LSORT_ROOT_B=1024 python tools/ab_total.py --dists lognormal2:5e8,normal:1e8 --reps 4 > gpurun_out/s3_ab_root1024.log 2>&1
LSORT_ROOT_B=256 python tools/ab_total.py --dists lognormal2:5e8,normal:1e8 --reps 4 > gpurun_out/s3_ab_root256.log 2>&1
LSORT_TRACE=1 python tools/profile_sort.py uniform 10000000 3 > gpurun_out/s3_trace_c1.log 2>&1
