mkdir -p gpurun_out
for v in 0 2 3; do FOLD_DBG_FWD=$v timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke_$v.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$v.log; done
