# compute-sanitizer over one solve + loss + backward (the wavefront sweep's
# cross-CTA mailbox / progress protocols, the dataflow adjoint), 128^2 and 256^2
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python scripts/prof_solve.py ${SAN_N:-128} > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.log
done
