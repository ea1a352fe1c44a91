set -x
for c in 0 2 4 6; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo bench$c $?; done
