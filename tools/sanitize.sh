#!/bin/bash
# compute-sanitizer over every kernel family; logs in gpurun_out/
# usage: tools/sanitize.sh [tool ...]   (default: memcheck racecheck synccheck initcheck)
tools=${@:-memcheck racecheck synccheck initcheck}
for t in $tools; do
  for f in tma reg persist csr sorted ic0 peer order; do
    echo "== $t $f" >> gpurun_out/r02_sanitize_$t.txt
    timeout 900 compute-sanitizer --tool $t --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_target.py $f >> gpurun_out/r02_sanitize_$t.txt 2>&1
    echo "rc=$?" >> gpurun_out/r02_sanitize_$t.txt
  done
done
