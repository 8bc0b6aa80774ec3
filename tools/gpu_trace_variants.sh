# Backward diagnostics: per-tile timelines (FOLD_DBG_BWD) for each entry of
# $VARIANTS = "name:LIB:ENV=.. ;..." (LIB = a tools/build_variant.sh name or "base"), C3 and C4 B=1024
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-base:base:}"
for v in "${VS[@]}"; do
  name=${v%%:*}; rest=${v#*:}; lib=${rest%%:*}; envs=${rest#*:}
  L=""; [ "$lib" != base ] && L="FOLD_LIB_PATH=paper_1702_02181_b200/_lib_variants/$lib/libfold.so"
  for c in ${CONFIGS:-c3 c4}; do
    env $L $envs FOLD_DBG_BWD=1 timeout 300 python tools/trace_bwd.py --config $c --batch 1024 --levels 4 > gpurun_out/trace_bwd_${c}_$name.txt 2>&1
    echo "== $name $c"; sed -n 2p gpurun_out/trace_bwd_${c}_$name.txt
  done
done
