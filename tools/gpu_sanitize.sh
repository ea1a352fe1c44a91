set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 600 python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo plain $?
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py > gpurun_out/san_$t.log 2>&1; echo $t $?
done
