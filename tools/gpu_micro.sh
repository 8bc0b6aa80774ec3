O=gpurun_out/micro; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1702_02181_b200/csrc tools/micro/l2_ingress.cu -o /tmp/l2_ingress -lcuda 2>/dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1702_02181_b200/csrc tools/micro/mma_contention.cu -o /tmp/mma_contention -lcuda 2>/dev/null
timeout 120 /tmp/l2_ingress > $O/l2_ingress.json 2>&1
timeout 300 /tmp/mma_contention > $O/mma_contention.json 2>&1
cat $O/*.json
