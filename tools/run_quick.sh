# quick GPU pass: gpu tests + per-op kernel times (usage: bash tools/run_quick.sh TAG [prof targets])
TAG=$1; shift
O=gpurun_out; mkdir -p $O
[ -z "$NO_TESTS" ] && timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_tests.log 2>&1; echo rc=$? >> $O/${TAG}_tests.log
timeout 600 python tools/prof_ops.py ${@:-c3} > $O/${TAG}_prof.log 2>&1
