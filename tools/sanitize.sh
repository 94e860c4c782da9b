#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the hot
# kernels (tools/sanitize_drive.py); logs to gpurun_out/sanitize_<tool>_<part>.log
mkdir -p gpurun_out
for part in psh pool backbone; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_drive.py $part \
      > gpurun_out/sanitize_${tool}_${part}.log 2>&1
    echo "exit $?" >> gpurun_out/sanitize_${tool}_${part}.log
    echo "$tool $part: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|exit' gpurun_out/sanitize_${tool}_${part}.log | tr '\n' ' ')"
  done
done
