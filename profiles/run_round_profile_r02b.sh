#!/bin/bash
# Round-2 (session 2) bundle, one gpurun call on 1 GPU:
#  0) the GPU parity suite
#  1) the default bench line (headline + cpu_baseline + e2e + L sweep)
#  2) ncu launch list of one full-batch fwd+bwd step at L=128 (--splits 1)
#  3) ncu --set full of the tcgen05 kernels of that step
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout=600 > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
K='regex:state_scan|fwd_parallel_kernel|fwd_fused_kernel|bwd_fused_kernel|bwd_parallel_kernel|gates_|mscan_kernel|assemble_kernel|qn_kernel|nscan_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "$K" -s 24 -c 8 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 > gpurun_out/launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on \
    -k 'regex:state_scan_kernel|fwd_fused_kernel|bwd_fused_kernel' -s 9 -c 3 \
    -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --splits 1 > gpurun_out/prof_full.log 2>&1
python profiles/ncu_top.py gpurun_out/prof_full.ncu-rep 12 > gpurun_out/prof_full.txt 2>&1
ls -la gpurun_out
