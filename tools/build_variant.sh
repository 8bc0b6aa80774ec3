# Build a variant libfold.so for A/B runs: tools/build_variant.sh NAME "-DMACRO ..."
# -> paper_1702_02181_b200/_lib_variants/NAME/libfold.so (git-ignored; travels with gpurun);
# select it with FOLD_LIB_PATH=paper_1702_02181_b200/_lib_variants/NAME/libfold.so
set -e
D=paper_1702_02181_b200/_lib_variants/$1
mkdir -p $D
FOLD_LIB_PATH=$PWD/$D/libfold.so FOLD_NVCC_EXTRA="$2" python -c "from paper_1702_02181_b200 import build; build.build(force=True)"
ls -la $D/libfold.so
