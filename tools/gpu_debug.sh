set -x
timeout 900 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build $?
timeout 150 python -X faulthandler -c "
import faulthandler, sys
faulthandler.dump_traceback_later(45, repeat=True, file=sys.stdout)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_dbg.log 2>&1; echo smoke $?
