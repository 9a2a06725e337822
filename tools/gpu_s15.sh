set -u
O=gpurun_out/s15
mkdir -p $O
B="python bench.py --config C5 --virtual-shards 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > $O/base.log 2>&1
PEEL_ESORT=0 timeout 600 $B > $O/noesort.log 2>&1
PEEL_BIN_ROUND_FRAC=0.01 timeout 600 $B > $O/frac01.log 2>&1
PEEL_BIN_ROUND_FRAC=0.04 timeout 600 $B > $O/frac04.log 2>&1
echo done > $O/done
