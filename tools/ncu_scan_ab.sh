#!/bin/bash
# ncu issue/stall metrics of the scan kernel for library variants: tools/ncu_scan_ab.sh TAG CONFIG lib1.so lib2.so ...
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
M="gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_no_instruction.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_not_selected.ratio,smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,smsp__average_warp_latency_issue_stalled_branch_resolving.ratio,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active"
for lib in "$@"; do
  name=$(basename $lib .so); L=""; [ "$lib" != "-" ] && L="SKS_LIB=$lib"; [ "$lib" = "-" ] && name=intree
  env $L timeout 900 ncu --metrics $M --clock-control none -k regex:scan2_kernel -c 1 --csv python tools/prof_step.py --config $CFG --steps 1 > $OUT/ncu_${name}.csv 2> $OUT/ncu_${name}.err
  python - $OUT/ncu_${name}.csv $name <<'PY'
import csv, sys, io
txt = open(sys.argv[1]).read()
lines = [l for l in txt.splitlines() if l.startswith('"')]
r = list(csv.DictReader(io.StringIO("\n".join(lines))))
print(sys.argv[2], {x["Metric Name"].replace("smsp__average_warp_latency_issue_stalled_", "stall_"): x["Metric Value"] for x in r})
PY
done
