# GPU tests, main bench legs and launch list + DRAM traffic after the elementwise-pass changes
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
timeout 600 python bench.py --no-cpu --no-c4 --no-ingest > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_ew.csv python tools/profile_step.py --steps 1 > /dev/null 2>&1
echo done
