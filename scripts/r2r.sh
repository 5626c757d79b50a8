#!/bin/bash
set -u
B=oracle/_ref/shimtests/ref_tests_b200
for args in "assembly | d|assembly | t" "assembly | d|assembly | s" "assembly | t|assembly | s" "assembly | s|assembly | c" "assembly | c|assembly | m" "assembly | m|assembly | g" "assembly | d|assembly | c" "assembly | t|assembly | c"; do
  IFS='|' read -ra A <<< "$(echo "$args" | sed 's/|assembly/|assembly/g')"
  a1="assembly |${args#assembly |}"; a1="${args%%|assembly*}"; a2="assembly${args#*|assembly}"
  out=$(timeout 300 $B "$a1" "$a2" 2>&1); rc=$?
  echo "rc=$rc [$a1] [$a2] :: $(echo "$out" | tail -1)"
done
