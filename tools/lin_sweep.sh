set -x
python tools/prof_linear.py bert_qkv bert_ffn1 bert_ffn2 llama_q llama_kv llama_up llama_down > gpurun_out/r2_lin_default.log 2>&1
for cfg in "1 256" "1 192" "1 128" "2 128" "2 256"; do set -- $cfg; MS_GEMM_CLUSTER=$1 MS_GEMM_BN=$2 python tools/prof_linear.py bert_qkv >> gpurun_out/r2_lin_sweep.log 2>&1; echo "^^ cl=$1 bn=$2" >> gpurun_out/r2_lin_sweep.log; done
ncu --set full --clock-control none --import-source on -k regex:umma_gemm -c 3 -o gpurun_out/r2_ncu_bert_qkv python tools/prof_linear.py bert_qkv > gpurun_out/r2_ncu_bert_qkv.log 2>&1
