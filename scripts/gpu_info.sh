# box info + both arithmetic modes of the default bench (scratch run)
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt; free -g >> gpurun_out/lscpu.txt
python bench.py --dtype f32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
