#!/bin/bash
# The RD_CHECKS debug build (device-side bounds assertions) over the GPU test suite and a few
# bench steps of every config: bash tools/gpu_checks.sh <tag>
TAG=${1:-chk}
mkdir -p gpurun_out
python -m paper_2406_01467_b200.build --checks > gpurun_out/checks_build_$TAG.log 2>&1 || { echo "checks build failed"; exit 1; }
export RADE_LIB=$PWD/paper_2406_01467_b200/librade_checks.so
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/checks_pytest_$TAG.log 2>&1
echo "pytest (RD_CHECKS) rc=$?" | tee -a gpurun_out/checks_pytest_$TAG.log
tail -2 gpurun_out/checks_pytest_$TAG.log
for c in C3 C1 C2 C4; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/checks_bench_${c}_$TAG.log 2>&1
  echo "bench $c (RD_CHECKS) rc=$?" | tee -a gpurun_out/checks_pytest_$TAG.log
done
for c in C3; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --distortion --normal-consistency --k5 split > gpurun_out/checks_bench_${c}_reg_$TAG.log 2>&1
  echo "bench $c --distortion --normal-consistency --k5 split (RD_CHECKS) rc=$?" | tee -a gpurun_out/checks_pytest_$TAG.log
done
grep -h "RD_CHECK failed" gpurun_out/checks_*_$TAG.log | head -5
echo "RD_CHECK failures: $(grep -h "RD_CHECK failed" gpurun_out/checks_*_$TAG.log | wc -l)" | tee -a gpurun_out/checks_pytest_$TAG.log
