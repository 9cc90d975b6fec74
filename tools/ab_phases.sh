for d in normal uniform rootdups zipf; do echo "== $d"; python tools/profile_sort.py $d 100000000 4 2>&1 | tail -2; done
