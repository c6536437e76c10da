#!/bin/bash
# Round captures (run under gpurun, 1 GPU): for each workload the bench
# line, the per-launch ncu list (gpu__time_duration.sum, --clock-control
# none) and one `ncu --set full` capture of the hot kernel, exported to
# gpurun_out/ (raw / source / details pages); then the seam pass.
# usage: profiles/capture_all.sh <round tag, e.g. r1>
r=${1:-r1}
for w in config1 config2_p1 config2_p2 config2_p3 config2_p4; do
  bash profiles/run_prof.sh ${r}_$w --workload $w
done
KREGEX=k_seam_list bash profiles/run_prof.sh ${r}_config1_seams --workload config1
