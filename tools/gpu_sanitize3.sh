# compute-sanitizer on the split-K backward (k_bwd_levels k-half units + ring hand-over):
# C2 B=4 (256-row levels: 128-column split units), C3 B=64 at S=128 (many small split levels)
O=gpurun_out/san3; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for case in "c2 4 bf16" "c3 64 bf16 128"; do
    n=$(echo $case | tr ' ' '_')
    timeout 900 $CS --tool $tool --print-limit 10 python tools/sanitize_case.py $case > $O/${tool}_$n.log 2>&1
    echo "$tool $case exit $?" >> $O/summary.txt
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|repeat max" $O/${tool}_$n.log | tail -2 >> $O/summary.txt
  done
done
cat $O/summary.txt
