set -u
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_zinv.py > gpurun_out/o_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -8 gpurun_out/o_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_zinv.py > gpurun_out/o_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -8 gpurun_out/o_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_zinv.py > gpurun_out/o_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -5 gpurun_out/o_synccheck.log
