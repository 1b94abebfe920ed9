# A/B of two builds of liblbm19.so in alternating processes (same box, same command)
# usage: bash profiles/ab_lib.sh <dir with baseline liblbm19.so> <bench args...>
set -u
BASE=$1; shift
mkdir -p gpurun_out
cp paper_2108_13241_b200/_lib/liblbm19.so /tmp/lib_new.so
for r in 1 2; do
  cp $BASE/liblbm19.so paper_2108_13241_b200/_lib/liblbm19.so
  echo "base $(timeout 900 python bench.py --no-cpu --no-e2e "$@" | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])')" >> gpurun_out/ab_lib.txt
  cp /tmp/lib_new.so paper_2108_13241_b200/_lib/liblbm19.so
  echo "new  $(timeout 900 python bench.py --no-cpu --no-e2e "$@" | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])')" >> gpurun_out/ab_lib.txt
done
