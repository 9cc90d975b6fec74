# A/B: root model sample size (env LSORT_ROOT_SAMPLE_SHIFT: n >> shift, cap raised to 4 Mi)
for sh in 9 8 7; do
  echo "== shift $sh"
  LSORT_ROOT_SAMPLE_SHIFT=$sh python tools/ab_total.py --dists lognormal2:5e8,normal:1e8,mixgauss:2e8 --variants "rmi_sample_cap=4194304" --reps 5
done
