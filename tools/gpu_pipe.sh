mkdir -p gpurun_out
F="--no-cpu-baseline --no-table1 --no-batch1 --no-sweep"
for i in 1 2; do
timeout 300 python bench.py $F > gpurun_out/pipe_on_$i.json 2>&1
timeout 300 python bench.py $F --no-pipeline > gpurun_out/pipe_off_$i.json 2>&1
done
for cb in "c2 1" "c2 64" "c4 1" "c3 1024"; do set -- $cb
timeout 300 python bench.py --config $1 --batch $2 $F > gpurun_out/pipe_on_$1_$2.json 2>&1
timeout 300 python bench.py --config $1 --batch $2 $F --no-pipeline > gpurun_out/pipe_off_$1_$2.json 2>&1
done
