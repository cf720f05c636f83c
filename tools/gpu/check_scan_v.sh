# GPU tests, main bench legs and the step's launch list after a change to the scan stores
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
timeout 600 python bench.py --no-cpu --no-c4 --no-ingest > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_scanv.csv python tools/profile_step.py --steps 1 > /dev/null 2>&1
echo done
