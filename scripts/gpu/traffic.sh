mkdir -p gpurun_out
for w in config4 config5; do
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/r2k_${w}_traffic.csv python scripts/ncu_c4_path.py $w > gpurun_out/r2k_${w}_traffic.log 2>&1
echo "$w rc=$?"
done
