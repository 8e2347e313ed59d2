# scratch GPU call (edited per experiment)
mkdir -p gpurun_out
make -C paper_2605_20977_b200 clean > /dev/null; make -C paper_2605_20977_b200 -j16 TRACE=1 > /dev/null 2>&1; echo build rc=$?
timeout 300 python tools/gemm_trace.py step_wq step_wo step_gu step_wd ch_mix ch_gu ch_d ch_head1 ch_head2 2>&1 | grep -v "^ *\(setup\|tma_issued\)"
