# compute-sanitizer on the round-2 kernels: MO path (schedule, grouped GEMMs, push-gather),
# CTA-pair TF32 GEMMs (FP32 mode at a size that uses them), converged-warp MMA issue (BF16)
O=gpurun_out/san2; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/mo_case.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import foldgen
from paper_1702_02181_b200 import fold_mo
prec = sys.argv[1]
T = foldgen.mo_table_c6(S0=64, S1=32, vocab=300)
gr = foldgen.mo_batch_c6(24, table=T)
params = foldgen.make_mo_params(T)
t = lambda x: torch.tensor(np.ascontiguousarray(x, np.int32).reshape(-1), device="cuda")
s = fold_mo.schedule(T, t(gr.op), t(gr.child), t(gr.token), t(gr.root))
model = fold_mo.MoModel([tuple(torch.tensor(x, device="cuda") for x in blk) for blk in params], prec)
h, acts = fold_mo.forward(s, model)
g1 = fold_mo.backward(s, model, acts, torch.tensor(foldgen.make_mo_upstream(gr.n_graphs, T), device="cuda"))
g2 = fold_mo.backward(s, model, acts, torch.tensor(foldgen.make_mo_upstream(gr.n_graphs, T), device="cuda"))
torch.cuda.synchronize()
print("mo_case", prec, "repeat max|diff|", max(float((a - b).abs().max()) for x, y in zip(g1, g2) for a, b in zip(x, y)))
PY
for tool in memcheck racecheck synccheck; do
  for case in "mo fp32" "mo tf32" "c2 8 fp32" "c2 4 bf16"; do
    n=$(echo $case | tr ' ' '_')
    if [ "${case%% *}" = "mo" ]; then cmd="python /tmp/mo_case.py ${case#* }"; else cmd="python tools/sanitize_case.py $case"; fi
    timeout 900 $CS --tool $tool --print-limit 10 $cmd > $O/${tool}_$n.log 2>&1
    echo "$tool $case exit $?" >> $O/summary.txt
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|repeat max" $O/${tool}_$n.log | tail -2 >> $O/summary.txt
  done
done
cat $O/summary.txt
