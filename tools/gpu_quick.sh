for g in 8 16; do
PSWA_BENCH_GOPS=$g timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-config5 --no-lrp > gpurun_out/bench_g$g.json 2> gpurun_out/bench_g$g.err
python -c "
import json; d=json.load(open('gpurun_out/bench_g$g.json'))
print($g, d['ms_per_frame'], d['config4_gop_batch'])"
done
