python -c "import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)"
timeout 600 python -m pytest tests/test_gpu_packed.py -x -q --tb=short 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_bk_check" -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "k_bk_check|dram__|gpu__time|lts__|ms_per" | head
