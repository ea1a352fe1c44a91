# ncu full captures of selected kernels (one bench step each); args: regex list
set -x
./tools/mb_warpchol > gpurun_out/mb.log 2>&1; echo mb $?
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/b1.json 2>gpurun_out/b1.err; echo b1 $?
i=0
for k in "$@"; do
  i=$((i+1))
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$k" --launch-skip 3 --launch-count 1 -o gpurun_out/prof_$i -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-measure-peak > gpurun_out/ncu_$i.log 2>&1; echo ncu$i $?
done
