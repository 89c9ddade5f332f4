#!/bin/bash
python -m paper_2203_08826_b200.build > /dev/null 2>&1 || exit 1
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__sass_inst_executed_op_ldgsts.sum,smsp__sass_inst_executed_op_shared_ld.sum,smsp__sass_inst_executed_op_shared_st.sum,smsp__sass_inst_executed_op_global_st.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed_op_branch.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_inst_executed_op_global_ld.sum,smsp__sass_thread_inst_executed.sum
QJ_TILE_CARRY=0 QJ_JIT_SKIP=ast ncu --metrics $M --clock-control none -k regex:qj_tile_jit -s 3 -c 1 --csv python tools/qft_passes.py 30 2 2>/dev/null | grep qj_tile | awk -F'","' '{print "qft1", $(NF-2), $NF}'
QJ_CIRC=h9 ncu --metrics $M --clock-control none -k regex:qj_tile_jit -s 1 -c 1 --csv python tools/qft_passes.py 30 2 2>/dev/null | grep qj_tile | awk -F'","' '{print "h9", $(NF-2), $NF}'
