#!/bin/bash
# Round-2 profiling pass (run on the GPU box via gpurun): per config, the ncu
# launch list of 2 steps of the product arm and one `ncu --set full` capture of
# the bench's dominant memsave op (NVTX-marked by tools/prof_step.py --mark).
cd "$(dirname "$0")/.."
OUT=gpurun_out
declare -A OP GEOM
OP[bert]=linear_fwd;      GEOM[bert]='{"M": 32768, "N": 768, "K": 768}'
OP[bertdx]=linear_dx;     GEOM[bertdx]='{"M": 32768, "N": 768, "K": 768}'
OP[bertlda]=linear_dropout_add_fwd; GEOM[bertlda]='{"M": 32768, "N": 768, "K": 3072}'
OP[resnet18]=conv2d_bn_fwd; GEOM[resnet18]='{"x": [256, 64, 56, 56], "w": [64, 64, 3, 3], "stride": [1, 1], "pad": [1, 1]}'
OP[resnet101]=conv2d_bn_dx; GEOM[resnet101]='{"x": [128, 1024, 14, 14], "w": [256, 1024, 1, 1], "stride": [1, 1], "pad": [0, 0]}'
OP[vgg16]=conv2d_dw;  GEOM[vgg16]='{"x": [128, 512, 28, 28], "w": [512, 512, 3, 3], "stride": [1, 1], "pad": [1, 1]}'
OP[vgg16c11]=conv2d_bn_fwd;  GEOM[vgg16c11]='{"x": [128, 3, 224, 224], "w": [64, 3, 3, 3], "stride": [1, 1], "pad": [1, 1]}'
OP[fig1]=conv2d_fwd;      GEOM[fig1]='{"x": [32, 8, 256, 256], "w": [8, 8, 3, 3], "stride": [1, 1], "pad": [1, 1]}'
OP[llama]=linear_fwd;     GEOM[llama]='{"M": 4096, "N": 14336, "K": 4096}'
OP[r101bn]=bn_add_relu_bwd; GEOM[r101bn]='{"shape": [128, 1024, 14, 14]}'
OP[r101bnf]=bn_relu_fwd; GEOM[r101bnf]='{"shape": [128, 1024, 14, 14]}'
for c in ${CONFIGS:-bert resnet18 resnet101 vgg16 fig1 llama r101bn r101bnf}; do
  cfg=$c; [[ $c == r101bn* ]] && cfg=resnet101; [[ $c == vgg16c11 ]] && cfg=vgg16
  [[ $c == bert?* ]] && cfg=bert
  if [[ $c != r101bn* && $c != vgg16c11 && $c != bert?* ]]; then
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
      --csv --log-file $OUT/r2_launches_$c.csv python tools/prof_step.py --config $cfg --steps 2 \
      > $OUT/r2_launches_$c.log 2>&1
  fi
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    --nvtx --nvtx-include "dominant/" -c 4 -f -o $OUT/r2_ncu_$c \
    python tools/prof_step.py --config $cfg --steps 1 --mark ${OP[$c]} --mark-geom "${GEOM[$c]}" \
    > $OUT/r2_ncu_$c.log 2>&1
  # keep the summaries, not the (large) report
  ncu -i $OUT/r2_ncu_$c.ncu-rep --page raw --csv > $OUT/r2_ncu_${c}_raw.csv 2>/dev/null
  ncu -i $OUT/r2_ncu_$c.ncu-rep --page details --csv > $OUT/r2_ncu_${c}_details.csv 2>/dev/null
  rm -f $OUT/r2_ncu_$c.ncu-rep
done
