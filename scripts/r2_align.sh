#!/bin/bash
# alignment of W / staging / gsum inside the symmetric buffer: 256 B vs 2 MiB (A/B at N=2 and N=4)
mkdir -p gpurun_out
bash scripts/mgpu_env_sweep2.sh 2 "CDSGD_P2P_ALIGN=256" "CDSGD_P2P_ALIGN=2097152" "CDSGD_P2P_ALIGN=256" "CDSGD_P2P_ALIGN=2097152" 2>&1 | tee gpurun_out/r2al_ab_n2.txt
bash scripts/mgpu_env_sweep2.sh 4 "CDSGD_P2P_ALIGN=256" "CDSGD_P2P_ALIGN=2097152" "CDSGD_P2P_ALIGN=256" "CDSGD_P2P_ALIGN=2097152" 2>&1 | tee gpurun_out/r2al_ab_n4.txt
