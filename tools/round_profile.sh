#!/bin/bash
# One gpurun call: single-launch ncu --set full captures of the dense pass (c3, c4), the symmetric
# pass (c3) and both block-sparse passes (c3 size, p = 0.5 gather / p = 0.9 slab), exported on the
# box to CSV pages (raw, details, source) and summarised (the .ncu-rep files are ~25 MB each and
# are deleted: gpurun copies back at most 64 MiB); then the bench lines (c3 with variants, c4, c2,
# reference arm), the bench launch list, kernel-side shard scaling and small-config latency.
# Usage: bash tools/round_profile.sh r02
set -u
R=$1
O=gpurun_out
mkdir -p $O
cap() {   # cap <tag> <kernel regex> <skip> <command...>
  local tag=$1 k=$2 sk=$3; shift 3
  "$@" > $O/pt_${R}_$tag.log 2>&1 || { echo "plain run failed: $tag"; return; }
  ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 -o $O/prof_${R}_$tag "$@" \
      > $O/ncu_${R}_$tag.log 2>&1
  ncu -i $O/prof_${R}_$tag.ncu-rep --page raw --csv > $O/${R}_${tag}_full_raw.csv 2>/dev/null
  ncu -i $O/prof_${R}_$tag.ncu-rep --page details --csv > $O/${R}_${tag}_details.csv 2>/dev/null
  ncu -i $O/prof_${R}_$tag.ncu-rep --page source --csv --print-source sass > $O/${R}_${tag}_source.csv 2>/dev/null
  gzip -f $O/${R}_${tag}_source.csv
  python tools/ncu_summary.py $tag=$O/prof_${R}_$tag.ncu-rep > $O/${R}_${tag}_summary.json 2>&1
  rm -f $O/prof_${R}_$tag.ncu-rep
}
cap c3 panel_kernel 3 python tools/prof_target.py c3
cap c4 wide_tc_kernel 3 python tools/prof_target.py c4
NSRGS_NARROW_TC=0 cap c4cc panel_kernel 3 python tools/prof_target.py c4
cap c3sym sym_block 3 python tools/prof_target.py c3 sym
cap w25 wide_tc_kernel 3 python tools/prof_target.py w25
cap w16 wide_tc_kernel 3 python tools/prof_target.py w16
cap c3bsr bsr_kernel 5 python tools/bsr_bench.py 20000 5 0.5 4
cap c3bsrslab bsr_slab 5 python tools/bsr_bench.py 20000 5 0.9 4
python bench.py > $O/bench_$R.log 2>&1
python bench.py --config c4 --no-sym-variant --side-configs "" > $O/bench_${R}_c4.log 2>&1
NSRGS_NARROW_TC=0 python bench.py --config c4 --no-sym-variant --no-bsr-variant --no-cpu-baseline --side-configs "" > $O/bench_${R}_c4_cudacore.log 2>&1
python bench.py --config c2 --no-bsr-variant > $O/bench_${R}_c2.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_${R}_reference.log 2>&1
L="--steps 1 --warmup 3 --no-sym-variant --no-bsr-variant --no-cpu-baseline --no-read-probe"
python bench.py $L > $O/plain_bench_$R.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_${R}_c3.csv \
    python bench.py $L > $O/ncu_launches_$R.log 2>&1
if [ "${SKIP_EXTRA:-0}" = "0" ]; then
  python tools/shard_scaling.py c3 > $O/shard_${R}.json 2>&1
  python tools/shard_scaling.py c4 >> $O/shard_${R}.json 2>&1
  python tools/coop_ab.py c1,c2 > $O/latency_${R}.log 2>&1
fi
echo done
