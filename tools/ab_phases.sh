# per-phase A/B of the sort on the BASELINE distributions (1e8 keys):
#   bash tools/ab_phases.sh [ENV=VALUE ...]  (e.g. LSORT_NO_FWD=1)
for d in normal uniform lognormal05 rootdups zipf; do echo "== $d $*"; env "$@" python tools/profile_sort.py $d 100000000 4 2>&1 | tail -2; done
