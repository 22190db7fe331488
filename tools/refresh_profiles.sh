# Round-end evidence refresh on the GPU box (gpurun): full GPU suite, smoke, bench line,
# bench launch list, ncu full capture of the sweep kernels, all five configs.
mkdir -p gpurun_out
set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-modes --no-plain > gpurun_out/ncu_bench.log 2>&1; tail -c 100 gpurun_out/ncu_bench.log
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_stream|k_finalize" -s 20 -c 2 -o gpurun_out/stream_rmat24_reduced_warm python tools/step_once.py 4 reduced > gpurun_out/ncu_stream.log 2>&1; tail -1 gpurun_out/ncu_stream.log
timeout 1500 python tools/all_configs.py > gpurun_out/all_configs.json 2> gpurun_out/all_configs.err; tail -c 200 gpurun_out/all_configs.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -c 300 gpurun_out/bench_reference.json
timeout 600 python tools/shard_scaling.py 4 1 2 4 8 local > gpurun_out/shard_scaling_local.json 2> gpurun_out/shard_scaling_local.err
PRGPU_PROFILE=2 timeout 300 python tools/profile_create_sharded.py 4 8 0 > gpurun_out/create_sharded_profile.log 2>&1
PRGPU_PROFILE=2 timeout 300 python tools/time_create.py 4 2 > gpurun_out/create_profile.log 2>&1
