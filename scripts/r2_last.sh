#!/bin/bash
# last driver-like pass at the final commit on a 4-GPU box: GPU suite + smoke + N=1 arms, then N=2/N=4 bench
TAG=r2z bash scripts/r2_final_n1.sh
TAG=r2z bash scripts/r2_final_mgpu.sh
