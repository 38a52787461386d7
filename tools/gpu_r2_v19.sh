cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_driver.py tiny small_multi odd midsplit fused klexact lmhead > gpurun_out/r02_sanitize_initcheck_nolmupdate.log 2>&1; echo "initcheck (all but lmupdate) rc=$?"; tail -2 gpurun_out/r02_sanitize_initcheck_nolmupdate.log
timeout 1200 compute-sanitizer --tool initcheck --print-limit 1000000 python tools/sanitize_driver.py lmupdate > gpurun_out/r02_sanitize_initcheck_lmupdate_full.log 2>&1; echo "initcheck lmupdate rc=$?"
grep "^=========     at " gpurun_out/r02_sanitize_initcheck_lmupdate_full.log | sed 's/+0x.*//' | sort | uniq -c > gpurun_out/r02_sanitize_initcheck_lmupdate_kernels.txt; cat gpurun_out/r02_sanitize_initcheck_lmupdate_kernels.txt
rm -f gpurun_out/r02_sanitize_initcheck_lmupdate_full.log
