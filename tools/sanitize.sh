#!/bin/bash
# compute-sanitizer runs of every decode variant on small seeded launches; logs to gpurun_out/.
#   bash tools/sanitize.sh [tag]
tag=${1:-r2}
out=gpurun_out/sanitize_$tag
mkdir -p $out
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
timeout 1800 $CS --tool racecheck --racecheck-report all python tools/sanitize_driver.py > $out/racecheck.log 2>&1
echo "racecheck rc $?" | tee -a $out/summary.txt
timeout 1800 $CS --tool synccheck python tools/sanitize_driver.py > $out/synccheck.log 2>&1
echo "synccheck rc $?" | tee -a $out/summary.txt
timeout 1200 $CS --tool memcheck --leak-check no python tools/sanitize_driver.py > $out/memcheck.log 2>&1
echo "memcheck rc $?" | tee -a $out/summary.txt
timeout 600 $CS --tool memcheck python tools/sanitize_driver.py --errors > $out/memcheck_errors.log 2>&1
echo "memcheck_errors rc $?" | tee -a $out/summary.txt
timeout 1200 $CS --tool initcheck python tools/sanitize_driver.py --case v1_deg6 v2_deg18 v7_long > $out/initcheck.log 2>&1
echo "initcheck rc $?" | tee -a $out/summary.txt
