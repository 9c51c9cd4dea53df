#!/bin/bash
# One parametrized runner for gpurun calls (replaces the single-use r*.sh
# scripts of round 1).  Usage, from the repo root on the GPU box:
#   bash tools/gpu_suite.sh TAG STEP [STEP ...]
# STEP is one of
#   build                 __graft_entry__.build()
#   smoke                 __graft_entry__.smoke()
#   tests[:EXPR]          pytest -m gpu (optionally -k EXPR)
#   file:PATH             pytest -m gpu on one test file
#   bench[:ARGS]          python bench.py ARGS  (ARGS with commas for spaces)
#   ref[:ARGS]            python bench.py --impl reference ARGS
#   launches[:ARGS]       ncu launch list of bench.py (gpu__time_duration, --clock-control none)
#   ncu:KERNEL_REGEX:ARGS one `ncu --set full` capture of a kernel of tools/profile_target.py ARGS
#   py:SCRIPT[:ARGS]      python SCRIPT ARGS
# Logs go to gpurun_out/TAG_*.
TAG=$1; shift
mkdir -p gpurun_out
for STEP in "$@"; do
  KIND=${STEP%%:*}; REST=${STEP#*:}; [ "$REST" = "$STEP" ] && REST=""
  ARGS=${REST//,/ }
  case $KIND in
    build) python -c "import __graft_entry__ as g; g.build(); print('build ok')" > gpurun_out/${TAG}_build.log 2>&1; tail -1 gpurun_out/${TAG}_build.log ;;
    smoke) python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log ;;
    tests) if [ -n "$REST" ]; then K=(-k "$ARGS"); else K=(); fi
           timeout 2400 python -m pytest tests -q -m gpu -x "${K[@]}" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log ;;
    file) timeout 1800 python -m pytest $ARGS -q -m gpu > gpurun_out/${TAG}_$(basename ${ARGS%% *} .py).log 2>&1; echo "file rc=$?"; tail -3 gpurun_out/${TAG}_$(basename ${ARGS%% *} .py).log ;;
    bench) timeout 1800 python bench.py $ARGS > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/${TAG}_bench.err | cut -c1-400 ;;
    ref) timeout 900 python bench.py --impl reference $ARGS > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?" ;;
    launches) timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py $ARGS > gpurun_out/${TAG}_launches.log 2>&1; echo "launches rc=$?" ;;
    ncu) KRE=${REST%%:*}; PA=${REST#*:}; PA=${PA//,/ }
         timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 1 -o gpurun_out/${TAG}_ncu -f python tools/profile_target.py $PA > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/${TAG}_ncu.log ;;
    py) SCRIPT=${REST%%:*}; PA=${REST#*:}; [ "$PA" = "$REST" ] && PA=""; PA=${PA//,/ }
        timeout 1800 python $SCRIPT $PA > gpurun_out/${TAG}_$(basename $SCRIPT .py).log 2>&1; echo "py $SCRIPT rc=$?"; tail -3 gpurun_out/${TAG}_$(basename $SCRIPT .py).log | cut -c1-600 ;;
    *) echo "unknown step $STEP" ;;
  esac
done
