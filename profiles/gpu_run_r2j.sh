timeout 600 python -m pytest tests/test_gpu_bucket.py -x -q --tb=short 2>&1 | tail -5
for v in default minb2; do
  if [ $v = minb2 ]; then export GWCP_B200_LIB=$PWD/variants/lib_minb2.so; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_j_$v.json 2> gpurun_out/bench_j_$v.err; tail -3 gpurun_out/bench_j_$v.err; python -c "
import json; d=json.load(open('gpurun_out/bench_j_$v.json')); print('$v', d['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_ms_eager'], d['run']['report_digest']==d['run']['report_digest_expected'])"
done
