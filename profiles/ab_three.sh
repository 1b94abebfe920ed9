# A/B/C of three library builds (abl/base.so, abl/new48.so, abl/new64.so) on one bench command
set -u
mkdir -p gpurun_out
for r in 1 2; do
  for b in base new48 new64; do
    cp abl/$b.so paper_2108_13241_b200/_lib/liblbm19.so
    echo "$b $(timeout 900 python bench.py --no-cpu --no-e2e "$@" | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), round(d["roofline"]["frac"],4))')" >> gpurun_out/ab3.txt
  done
done
