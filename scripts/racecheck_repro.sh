#!/usr/bin/env bash
# Known-correct minimal programs with the library's two racecheck-reported patterns
# (tests/helpers/racecheck_repro.cu), run plain and under racecheck.
O=gpurun_out/${1:-rc}; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o $O/rc_repro tests/helpers/racecheck_repro.cu
$O/rc_repro > $O/rc_repro_plain.log 2>&1; echo plain=$?
timeout 300 compute-sanitizer --tool racecheck --racecheck-report all $O/rc_repro > $O/rc_repro_racecheck.log 2>&1; echo racecheck=$?
cat $O/rc_repro_plain.log; tail -20 $O/rc_repro_racecheck.log
timeout 1200 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_racecheck_smoke.log 2>&1; echo rc_smoke=$?
tail -3 $O/sanitizer_racecheck_smoke.log
timeout 1200 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_memcheck_smoke.log 2>&1; echo mc_smoke=$?
tail -3 $O/sanitizer_memcheck_smoke.log
timeout 1200 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_synccheck_smoke.log 2>&1; echo sc_smoke=$?
tail -3 $O/sanitizer_synccheck_smoke.log
