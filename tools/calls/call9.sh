set -x
nproc; python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; tail -c 3000 gpurun_out/bench_cfg1.json
( time BENCH_NO_SINGLE_THREAD=1 python bench.py --impl reference --steps 2 --warmup 1 ) > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 1500 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
