#!/bin/bash
# GPU-box evidence pass, split so that each gpurun call runs at most one ncu:
#   bash tools/round_profile.sh TAG CONFIG bench  -> bench line (+ reference arm) and the
#                                                    ncu launch list of the bench command
#   bash tools/round_profile.sh TAG CONFIG full   -> one ncu --set full capture of a
#                                                    steady-state step (3 kernels x 3 sweeps)
set -u
TAG=$1
CFG=${2:-c1}
MODE=${3:-bench}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ "$MODE" = bench ]; then
  python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err || { tail -20 $OUT/bench.err; exit 1; }
  python bench.py --config $CFG --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
  python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
      python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu > $OUT/ncu_launch.log 2>&1
  tail -c 600 $OUT/bench.json
else
  python tools/exp/step_run.py $CFG 4 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_synthesis|k_ring|k_analysis" \
      --launch-skip 9 --launch-count 9 -o $OUT/prof python tools/exp/step_run.py $CFG 4 > $OUT/ncu_full.log 2>&1
  tail -3 $OUT/ncu_full.log
fi
