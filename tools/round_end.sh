#!/bin/bash
# Full GPU validation + bench lines of every config (run on the GPU box via gpurun).
cd "$(dirname "$0")/.."
OUT=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:randomly > $OUT/gputest.log 2>&1; echo "pytest rc=$?" >> $OUT/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
for c in ${CONFIGS:-bert resnet18 resnet101 vgg16 fig1 llama}; do
  timeout 900 python bench.py --config $c > $OUT/r2_bench_$c.log 2>&1
  tail -1 $OUT/r2_bench_$c.log > $OUT/r2_bench_$c.json
done
timeout 600 python bench.py --impl reference > $OUT/r2_bench_reference.log 2>&1
tail -1 $OUT/r2_bench_reference.log > $OUT/r2_bench_reference_arm.json
