bash scripts/gpu_ncu.sh gpt24
bash scripts/gpu_ncu.sh unet
