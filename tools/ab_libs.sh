#!/bin/bash
# A/B of two builds of the C-ABI library on one GPU box (box-to-box variance is
# larger than most kernel changes): put the builds at abtest/libA.so and
# abtest/libB.so (git-ignored), then run under gpurun
#   bash tools/ab_libs.sh "python tools/prof_conv.py layer1_fwd" [rounds]
# Each round runs the command once per build, alternating A and B.
cd "$(dirname "$0")/.."
L=paper_2404_12406_b200/libmemsave_b200.so
cp $L abtest/cur.so
for round in $(seq 1 ${2:-3}); do
  for v in A B; do
    cp abtest/lib$v.so $L
    echo "$v $round $(bash -c "$1" 2>&1 | tr '\n' ' ')"
  done
done
cp abtest/cur.so $L
rm -f abtest/cur.so
