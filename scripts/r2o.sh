#!/bin/bash
set -u
for c in "config names" "unit cube" "triangle" "annihilates" "scaled weights" "quadrature scaled" "mass action" "action integrand" "actions match" "batched action" "engines agree" "numerically symmetric" "tightening" "mode guards" "discontinuous" "two cell" "shared entries" "coordinate" "mismatched" "global error" "continuous dofmap" "near-coincident"; do
  out=$(timeout 120 oracle/_ref/shimtests/ref_tests_b200 "$c" 2>&1); rc=$?
  echo "rc=$rc case=$c :: $(echo "$out" | tail -1)"
done
