# T5: compute-sanitizer memcheck / racecheck / synccheck on small cases of every
# kernel family (BF16 tcgen05 wide + narrow kernels, TF32/3xTF32 GEMMs, scheduler, SST) +
# the L2 ingress microbenchmark. Outputs in gpurun_out/san/.
O=gpurun_out/san; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1702_02181_b200/csrc tools/micro/l2_ingress.cu -o /tmp/l2_ingress -lcuda 2>/dev/null
timeout 120 /tmp/l2_ingress > $O/l2_ingress.json 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for case in "c1 8 fp32" "c1 8 bf16" "c2 4 bf16" "c2 2 fp32" "c3 16 bf16 300" "c3 16 tf32 300" "c4 2 bf16" "sst 8 fp32"; do
    n=$(echo $case | tr ' ' '_')
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_case.py $case > $O/${tool}_$n.log 2>&1
    echo "$tool $case exit $?" >> $O/summary.txt
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|sanitize_case" $O/${tool}_$n.log | tail -3 >> $O/summary.txt
  done
done
cat $O/summary.txt
