timeout 600 python -m pytest tests/test_gpu_bucket.py tests/test_gpu_packed.py tests/test_gpu_validate.py -x -q --tb=short 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; tail -3 gpurun_out/bench_m.err; python -c "
import json; d=json.load(open('gpurun_out/bench_m.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['kernel_ms_eager'], d['run']['report_digest']==d['run']['report_digest_expected'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_bk_check" -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "k_bk_check|dram__|gpu__time|lts__" | head
