mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_all.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/gpu_tests_all.log
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 exit $?"
timeout 600 python bench.py --config 2 --scheme eulerian > gpurun_out/bench_cfg2_eulerian.json 2> gpurun_out/bench_cfg2_eulerian.err; echo "eu exit $?"
timeout 300 python tools/probes/stream_overlap.py > gpurun_out/stream_overlap.log 2>&1; echo "probe $?"; cat gpurun_out/stream_overlap.log
