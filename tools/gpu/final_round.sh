# Round-end run: GPU tests, the default bench line, then the ncu launch list / traffic / captures
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
TAG=r02 timeout 1200 bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
echo done
