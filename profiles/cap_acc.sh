set -u
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for W in c4 c5; do
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python profiles/run_one.py --workload $W --repeat 1 > gpurun_out/ncu_l_$W.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_access" -c 1 \
  -o gpurun_out/acc_$W python profiles/run_one.py --workload $W --repeat 1 > gpurun_out/ncu_f_$W.log 2>&1
ncu -i gpurun_out/acc_$W.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/acc_${W}_src.csv 2>&1
ncu -i gpurun_out/acc_$W.ncu-rep --page details --csv > gpurun_out/acc_${W}_details.csv 2>&1
rm -f gpurun_out/acc_$W.ncu-rep
done
ls -la gpurun_out
