# compute-sanitizer memcheck / racecheck / initcheck over scripts/sanitize.py; logs into gpurun_out/$1
O=gpurun_out/${1:-sanitize}
mkdir -p $O
for t in memcheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize.py > $O/sanitize_$t.txt 2>&1
  echo "$t rc=$?" >> $O/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize target ok" $O/sanitize_$t.txt >> $O/sanitize_summary.txt
done
cat $O/sanitize_summary.txt
