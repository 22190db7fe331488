mkdir -p gpurun_out/s3
timeout 1400 python -m pytest tests -m gpu -q -x > gpurun_out/s3/pytest_gpu.log 2>&1; tail -2 gpurun_out/s3/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1; tail -1 gpurun_out/s3/smoke.log
timeout 500 python bench.py > gpurun_out/s3/bench.json 2> gpurun_out/s3/bench.err; tail -c 300 gpurun_out/s3/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-modes --no-plain > gpurun_out/s3/ncu_bench.log 2>&1; tail -c 100 gpurun_out/s3/ncu_bench.log
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_stream|k_finalize" -s 20 -c 2 -o gpurun_out/s3/stream_rmat24_reduced_warm python tools/step_once.py 4 reduced > gpurun_out/s3/ncu_stream.log 2>&1; tail -1 gpurun_out/s3/ncu_stream.log
timeout 1500 python tools/all_configs.py > gpurun_out/s3/all_configs.json 2> gpurun_out/s3/all_configs.err; tail -c 200 gpurun_out/s3/all_configs.err
PRGPU_PROFILE=2 timeout 300 python tools/time_create.py 4 2 > gpurun_out/s3/create_profile.log 2>&1; tail -1 gpurun_out/s3/create_profile.log
