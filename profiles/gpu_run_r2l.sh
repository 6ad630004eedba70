timeout 1500 python -m pytest tests -x -q -m gpu --tb=short 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; tail -3 gpurun_out/bench_l.err; python -c "
import json; d=json.load(open('gpurun_out/bench_l.json')); print(d['ms_per_step'], d['e2e'], d['kernel_ms_eager'], d['run']['report_digest']==d['run']['report_digest_expected'])"
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bk_check" -c 1 -o gpurun_out/ncu/r2_c5_bkl python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bkl.log 2>&1; tail -2 gpurun_out/ncu_bkl.log
