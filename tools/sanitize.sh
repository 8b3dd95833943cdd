#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of tools/sanitize_run.py.  Output gpurun_out/$1/.
TAG=${1:-san}
O=gpurun_out/$TAG
mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 40 python tools/sanitize_run.py > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/rc.txt
  tail -4 $O/$tool.log
done
cat $O/rc.txt
