timeout 900 python -m pytest tests/test_gpu_bucket.py -x -q --tb=short 2>&1 | tail -3
for w in c5 c4; do GW_BUCKET=2 timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bk_$w.json 2> gpurun_out/bk_$w.err; tail -2 gpurun_out/bk_$w.err; python -c "
import json; d=json.load(open('gpurun_out/bk_$w.json')); print('$w', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], d['kernel_ms_eager'], d['run']['report_digest']==d['run'].get('report_digest_expected'))"; done
