cd $GRAFT_REPO_ROOT
for F in 1 12 45 64; do CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/gpu/dbg_tmap.py $F 2>&1 | tail -1; done
CVSR_SUBS=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/gpu/dbg_tmap.py 45 2>&1 | tail -1
CUDA_LAUNCH_BLOCKING=1 CVSR_LIB=build/variants/ch8.so timeout 120 python tools/gpu/dbg_tmap.py 45 2>&1 | tail -1
cuobjdump -sass -fun '_ZN4cvsr12k_layer_tmapILi6ELi2EEEvNS_7CodeDevENS_8DecStateEiif' paper_2108_08418_b200/libcvsr.so > gpurun_out/dbg_sass.txt 2>&1
