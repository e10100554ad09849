set -x
mkdir -p gpurun_out/r02
python bench.py --config cfg4 --json-out gpurun_out/r02/bench_cfg4.json > gpurun_out/r02/cfg4.out 2> gpurun_out/r02/cfg4.err; tail -c 600 gpurun_out/r02/cfg4.out; tail -3 gpurun_out/r02/cfg4.err
python bench.py --config cfg3 --steps 2 --warmup 1 --json-out gpurun_out/r02/bench_cfg3.json > gpurun_out/r02/cfg3.out 2> gpurun_out/r02/cfg3.err; tail -3 gpurun_out/r02/cfg3.err
python bench.py --config cfg2 --steps 3 --warmup 1 --json-out gpurun_out/r02/bench_cfg2.json > gpurun_out/r02/cfg2.out 2> gpurun_out/r02/cfg2.err; tail -3 gpurun_out/r02/cfg2.err
python bench.py --config cfg0 --steps 5 --warmup 3 --json-out gpurun_out/r02/bench_cfg0.json > gpurun_out/r02/cfg0.out 2> gpurun_out/r02/cfg0.err; tail -3 gpurun_out/r02/cfg0.err
