# compute-sanitizer passes (one tool per call; bounded by timeout): racecheck / synccheck /
# memcheck on smoke() (C1 n = 16 solve) and on fc_syev at N = 80 / 600 / 1000 (packed, 16-CTA
# cluster in shared memory, 16-CTA cluster with L2-resident columns)
tool=${1:-racecheck}
case=${2:-all}
set -x
timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --log-file gpurun_out/san_${tool}_${case}.log python tools/sanitize_case.py $case > gpurun_out/san_${tool}_${case}.out 2>&1
echo "exit $?" >> gpurun_out/san_${tool}_${case}.out
tail -5 gpurun_out/san_${tool}_${case}.log gpurun_out/san_${tool}_${case}.out
