# ncu evidence for every config (launch list + one --set full capture of the rollout kernel) and the critical-path kernel
for c in gpt24 unet gns16 llama80; do bash scripts/gpu_ncu.sh $c; done
bash scripts/gpu_ncu_cp.sh gpt24
