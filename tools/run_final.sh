# full round-end style pass: tests, smoke, bench (+ reference arm), launch list, ncu full of the hot kernels,
# per-config op timings and per-kernel breakdowns. usage: bash tools/run_final.sh TAG
TAG=$1
O=gpurun_out; mkdir -p $O
NCU='select_stream|project_stream|pos_slot|pos_copy|project_copy|sum_stream' NCU_SKIP=7 NCU_COUNT=7 bash tools/gpu_check.sh $TAG
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_ref.log 2>&1
timeout 900 python tools/bench_configs.py --reps 5 > $O/${TAG}_configs.jsonl 2> $O/${TAG}_configs.err
timeout 600 python tools/prof_ops.py c2 c3 c4 > $O/${TAG}_prof.log 2>&1
timeout 900 python tools/select_sweep.py --reps 3 > $O/${TAG}_select_sweep.jsonl 2> $O/${TAG}_select_sweep.err
