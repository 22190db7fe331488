# Evidence refresh without the full-size converged parity run (tools/refresh_s3.sh has it).
# Usage: bash tools/refresh_s3c.sh [outdir=gpurun_out/s3c]
O=${1:-gpurun_out/s3c}
mkdir -p $O
timeout 1400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 500 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-modes --no-plain > $O/ncu_bench.log 2>&1; tail -c 100 $O/ncu_bench.log
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_stream|k_finalize" -s 20 -c 2 -o $O/stream_rmat24_reduced_warm python tools/step_once.py 4 reduced > $O/ncu_stream.log 2>&1; tail -1 $O/ncu_stream.log
timeout 1500 python tools/all_configs.py > $O/all_configs.json 2> $O/all_configs.err; tail -c 200 $O/all_configs.err
