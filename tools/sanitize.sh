# compute-sanitizer over tools/sanitize_case.py: $1 = memcheck | racecheck | initcheck | synccheck
TOOL=${1:-memcheck}
O=gpurun_out/sanitize
mkdir -p $O
python tools/sanitize_case.py 32 mr > $O/plain.log 2>&1 || { echo "plain run failed"; tail -5 $O/plain.log; exit 1; }
tail -1 $O/plain.log
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 python tools/sanitize_case.py 32 mr > $O/$TOOL.log 2>&1
echo "exit $?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok |Error|hazard" $O/$TOOL.log | head -20
