cd $GRAFT_REPO_ROOT/scripts/ubench
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o finisher finisher.cu
for na in 1 2 3; do timeout 20 ./finisher $na; echo "rc=$?"; done 2>&1 | tee ../../gpurun_out/finisher.txt
