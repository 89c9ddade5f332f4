#!/bin/bash
# iterate: build, A/B probes (QJ_AB / QJ_WL), then the tile-path GPU tests
mkdir -p gpurun_out/it
python -m paper_2203_08826_b200.build > gpurun_out/it/build.log 2>&1 || { echo build failed; tail gpurun_out/it/build.log; exit 1; }
if [ -n "$QJ_AB" ]; then bash tools/ab_tile.sh 2>&1 | cut -c 1-1500; fi
if [ -n "$QJ_TESTS" ]; then
  timeout ${QJ_TEST_TIMEOUT:-1500} python -m pytest $QJ_TESTS -x -q > gpurun_out/it/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/it/pytest.log
fi
