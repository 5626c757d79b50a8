#!/bin/bash
set -u
for c in "kernels |" "assembly |" "mesh |" "kernels | a" "kernels | t" "kernels | m" "kernels | s" "kernels | e" "kernels | b" "kernels | p" "kernels | q" "kernels | u" "kernels | l" "kernels | c"; do
  out=$(timeout 300 oracle/_ref/shimtests/ref_tests_b200 "$c" 2>&1); rc=$?
  echo "rc=$rc case=$c :: $(echo "$out" | tail -1)"
done
