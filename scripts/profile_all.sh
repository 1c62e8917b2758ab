#!/bin/bash
# ncu captures of every config's dominant kernel from the current build (run
# under gpurun from the repo root; reports land in gpurun_out/, summarise them
# with scripts/ncu_summary.py).  Kernel replay for the deterministic runs;
# application replay for RCPSP120 (a node-limited search: kernel replay would
# carry the node reservations across passes).
set -x
export PYTHONPATH=$PWD
T=${1:-r02}
NCU="ncu --set full --clock-control none --import-source on -k regex:k_search"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_q14_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-tto --no-cpu-baseline > gpurun_out/${T}_launches.log 2>&1
$NCU -s 3 -c 1 -o gpurun_out/${T}_q14 python scripts/enum_one.py q14 > gpurun_out/${T}_prof.log 2>&1; gzip -9 gpurun_out/${T}_q14.ncu-rep
$NCU -s 3 -c 1 -o gpurun_out/${T}_csp python scripts/enum_one.py csp >> gpurun_out/${T}_prof.log 2>&1; gzip -9 gpurun_out/${T}_csp.ncu-rep
$NCU -s 1 -c 1 -o gpurun_out/${T}_r30s7 python scripts/solve_one.py 30 7 >> gpurun_out/${T}_prof.log 2>&1; gzip -9 gpurun_out/${T}_r30s7.ncu-rep
$NCU --replay-mode application -s 1 -c 1 -o gpurun_out/${T}_r120 python scripts/solve_one.py 120 1 0 1000000 >> gpurun_out/${T}_prof.log 2>&1; gzip -9 gpurun_out/${T}_r120.ncu-rep
