# failure rate of one fuzz case under scheduling toggles (each run a fresh process)
C=${1:-clusters:201660944:383816745:2}; R=${2:-6}
for env in "X=1" "LSORT_NO_PDL=1" "LSORT_BASE_SERIAL=1" "CUDA_LAUNCH_BLOCKING=1" "LSORT_NO_PDL=1 LSORT_BASE_SERIAL=1"; do
  f=0
  for i in $(seq $R); do
    env $env python tools/fuzz_sort.py --case $C > /tmp/rp.log 2>&1 || { f=$((f+1)); tail -n 1 /tmp/rp.log | cut -c1-200; }
  done
  echo "== $env: $f / $R failed"
done
