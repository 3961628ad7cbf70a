# ncu --set full of one kernel (regex $KREGEX) in tools/run_once.py; plain run first (B200_PROFILING.md)
CMD="python tools/run_once.py ${RUN_ARGS}"
$CMD > gpurun_out/plain_full.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -c ${KCOUNT:-1} -o gpurun_out/prof_${KNAME} $CMD > gpurun_out/ncu_full_${KNAME}.log 2>&1; echo ncu=$?; tail -3 gpurun_out/ncu_full_${KNAME}.log
