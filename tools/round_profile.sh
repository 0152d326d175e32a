#!/bin/bash
# One gpurun call: single-iteration ncu --set full of the dense pass (c3, c4) and of the
# symmetric pass (c3), the bench launch list, plus kernel-side shard scaling and small-config
# latency (no ncu).  Usage: bash tools/round_profile.sh r02
set -u
R=$1
mkdir -p gpurun_out
for c in c3 c4; do
  python tools/prof_target.py $c > gpurun_out/pt_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 3 -c 1 \
      -o gpurun_out/prof_${R}_$c python tools/prof_target.py $c > gpurun_out/ncu_${R}_$c.log 2>&1
done
python tools/prof_target.py c3 sym > gpurun_out/pt_c3sym.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sym_block -s 3 -c 1 \
    -o gpurun_out/prof_${R}_c3sym python tools/prof_target.py c3 sym > gpurun_out/ncu_${R}_c3sym.log 2>&1
python bench.py --steps 1 --warmup 3 --no-sym-variant > gpurun_out/plain_bench_$R.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${R}_c3.csv \
    python bench.py --steps 1 --warmup 3 --no-sym-variant > gpurun_out/ncu_launches_$R.log 2>&1
if [ "${SKIP_EXTRA:-0}" = "0" ]; then
  python tools/shard_scaling.py c3 > gpurun_out/shard_${R}.json 2>&1
  python tools/shard_scaling.py c4 >> gpurun_out/shard_${R}.json 2>&1
  python tools/coop_ab.py c1,c2 > gpurun_out/latency_${R}.log 2>&1
fi
echo done
