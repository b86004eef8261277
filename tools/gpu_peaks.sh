#!/bin/bash
# Measured FP32 FFMA peak (tools/ffma_peak.cu) with the SM clock sampled during the run.
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader -lms 100 > gpurun_out/peak_clocks.csv &
SMI=$!
sleep 0.3
for i in 1 2 3; do ./tools/ffma_peak.bin; done > gpurun_out/fp32_peak_runs.jsonl
kill $SMI
cat gpurun_out/fp32_peak_runs.jsonl
