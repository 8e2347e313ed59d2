# scratch GPU call (edited per experiment)
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-cpu --no-config4 --no-config5 --no-lrp"
P="import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_frame'], d['decoded_bit_exact'])"
timeout 600 $B 2>/dev/null | python -c "$P"
timeout 300 python tools/probe_ops.py 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 $B 2>/dev/null | python -c "$P"
