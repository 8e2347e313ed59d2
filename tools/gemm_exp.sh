# GEMM phase traces with the MMAs or the operand loads switched off (trace
# build; timing only): separates the TMA stream from the tensor pipe.
make -C paper_2605_20977_b200 clean all TRACE=1 > /dev/null 2>&1
for e in 0 1 2; do
  echo "=== GEMM_EXP $e"
  GEMM_EXP=$e timeout 300 python tools/gemm_trace.py ${OPS:-step_wo ch_mix step_wq ctx_ffn_gu}
done > gpurun_out/gemm_exp.txt 2>&1
