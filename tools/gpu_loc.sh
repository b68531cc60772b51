python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k "regex:k7_step|k8_fix" --csv --log-file gpurun_out/locality.csv python tools/locality_study.py > gpurun_out/locality.log 2>&1; echo "ncu rc=$?"
python tools/locality_study.py --summarise gpurun_out/locality.csv > gpurun_out/locality.md 2>&1; echo "sum rc=$?"
