# run the fuzz until it fails, then replay the failing case alone (plain, then LSORT_SYNC_DEBUG)
# usage: bash tools/fuzz_repro.sh SEED SECONDS DIST_FRACTION API_FRACTION
python tools/fuzz_sort.py --seconds ${2:-600} --seed ${1:-1} --dist ${3:-0} --api ${4:-0} > gpurun_out/fz.log 2>&1
rc=$?
tail -n 2 gpurun_out/fz.log | cut -c1-300
[ $rc -eq 0 ] && exit 0
line=$(grep "^FAIL\|^DIFF" gpurun_out/fz.log | head -n 1)
name=$(echo "$line" | awk '{print $2}' | sed 's/[@\/].*//')
n=$(echo "$line" | sed 's/.* n= *\([0-9]*\).*/\1/')
seed=$(echo "$line" | sed 's/.*seed= *\([0-9]*\).*/\1/')
flags=$(echo "$line" | sed 's/.*flags=\([0-9]*\).*/\1/')
world=$(echo "$line" | grep -o "world=[0-9]*" | sed 's/world=//')
[ -z "$world" ] && world=$(echo "$line" | grep -o "@[0-9]*" | sed 's/@//')
[ -z "$world" ] && world=0
api=$(echo "$line" | grep -o "api=[a-z]*" | sed 's/api=//')
[ -z "$api" ] && api=sort
C="$name:$n:$seed:$flags:$world:$api"
echo "replay $C"
for i in 1 2 3; do python tools/fuzz_sort.py --case $C 2>&1 | tail -n 1 | cut -c1-300; done
LSORT_SYNC_DEBUG=1 python tools/fuzz_sort.py --case $C 2>&1 | tail -n 3 | cut -c1-400
