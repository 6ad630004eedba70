timeout 600 python -m pytest tests/test_gpu_bucket.py -x -q --tb=short 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; tail -3 gpurun_out/bench_g.err; python -c "
import json; d=json.load(open('gpurun_out/bench_g.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_ms_eager'], d['run']['report_digest']==d['run']['report_digest_expected'])"
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bk_check" -c 1 -o gpurun_out/ncu/r2_c5_bkg python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bkg.log 2>&1; tail -2 gpurun_out/ncu_bkg.log
