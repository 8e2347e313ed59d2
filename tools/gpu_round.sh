# One GPU round: tests, smoke, per-probe ncu captures (the launches bench.py
# times for its kernel rooflines), bench, warm kernel times, launch list.
#   TAG=r02_sN bash tools/gpu_round.sh     (SKIP_TESTS=1, SKIP_NCU=1 to trim)
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
fi
NCU="ncu --set full --clock-control none --import-source on --profile-from-start off"
if [ -z "$SKIP_NCU" ]; then
timeout 1200 $NCU -f -o gpurun_out/ncu_probes python tools/profile_probes.py > gpurun_out/ncu_probes.log 2>&1; echo "ncu probes rc=$?"
# phase (t=1, g=1) of the entropy decoder, from a real decode (lane state advances per phase)
timeout 600 $NCU -f -k regex:decode_phase -s 5 -c 1 -o gpurun_out/ncu_decode_phase python tools/profile_decode.py > /dev/null 2>&1
python tools/ncu_traffic.py $TAG > gpurun_out/traffic.log 2>&1; echo "traffic rc=$?"; tail -2 gpurun_out/traffic.log
python tools/ncu_brief.py gpurun_out/ncu_decode_phase.ncu-rep > profiles/${TAG}_ncu_decode_phase.txt 2>&1
fi
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
PSWA_NO_PDL=1 PN=5 timeout 300 python tools/kernel_times.py > gpurun_out/kt.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/profile_decode.py > gpurun_out/ncu_launch.log 2>&1
ls gpurun_out
