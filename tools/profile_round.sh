#!/bin/bash
# Evidence for profiles/ (run on the GPU box from the repo root):
#   $1 = round tag (e.g. r2), $2 = config (cfg3 default)
# 1. bench line, 2. ncu launch list of a short bench run, 3. one ncu --set full
# capture of the dominant kernel (after the same program exited 0 without ncu).
set -u
tag=${1:-r2}; cfg=${2:-cfg3}
out=gpurun_out/prof_${tag}_${cfg}
mkdir -p $out
python bench.py --config $cfg --steps 1000 --warmup 10 > $out/bench.json 2> $out/bench.err || exit 1
python bench.py --config $cfg --steps 20 --warmup 3 --equil 200 --no-cpu-baseline > $out/short.json 2> $out/short.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $out/launches.csv \
  python bench.py --config $cfg --steps 20 --warmup 3 --equil 200 --no-cpu-baseline > $out/ncu_launch.log 2>&1
k=${3:-k_force}
ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 150 -c 1 \
  -o $out/force -f python bench.py --config $cfg --steps 20 --warmup 3 --equil 200 --no-cpu-baseline \
  > $out/ncu_full.log 2>&1
python tools/ncu_to_json.py $out/force.ncu-rep "$k" $cfg $out/ncu_force.json > /dev/null || true
python tools/ncu_summary.py $out/force.ncu-rep > $out/ncu_force_summary.txt 2>/dev/null || true
# gpurun brings back at most 64 MiB: keep the report only when asked to (KEEP_REP=1)
[ "${KEEP_REP:-0}" = 1 ] || rm -f $out/force.ncu-rep
echo done
