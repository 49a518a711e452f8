cd $GRAFT_REPO_ROOT
timeout 120 python scripts/m3_debug.py 65536 256 > gpurun_out/f_plain.log 2>&1; echo "rc=$?" >> gpurun_out/f_plain.log
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no python scripts/m3_debug.py 65536 256 > gpurun_out/f_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/f_memcheck.log
