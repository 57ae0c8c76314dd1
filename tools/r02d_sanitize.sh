# racecheck / synccheck / initcheck runs on small round trips
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --racecheck-report hazard python tools/sanitize_small.py decode > gpurun_out/r02_racecheck_decode.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r02_racecheck_decode.log
timeout 900 $CS --tool synccheck python tools/sanitize_small.py > gpurun_out/r02_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/r02_synccheck.log
timeout 900 $CS --tool initcheck python tools/sanitize_small.py decode > gpurun_out/r02_initcheck_decode.log 2>&1; echo "initcheck rc=$?" >> gpurun_out/r02_initcheck_decode.log
