#!/bin/bash
# one compute-sanitizer tool per gpurun call: TOOL=memcheck|racecheck
mkdir -p gpurun_out/san
python -m paper_2203_08826_b200.build > gpurun_out/san/build.log 2>&1 || exit 1
python tools/sanitize_driver.py > gpurun_out/san/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/san/plain.log; exit 1; }
timeout 900 compute-sanitizer --tool ${TOOL:-memcheck} --error-exitcode 3 python tools/sanitize_driver.py \
    > gpurun_out/san/${TOOL:-memcheck}.log 2>&1; echo "sanitizer ${TOOL:-memcheck} rc=$?"; tail -5 gpurun_out/san/${TOOL:-memcheck}.log
