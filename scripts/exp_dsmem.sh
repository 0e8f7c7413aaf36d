mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exp_dsmem scripts/exp_dsmem.cu && timeout 120 /tmp/exp_dsmem > gpurun_out/dsmem_gather.jsonl 2>&1
cat gpurun_out/dsmem_gather.jsonl
