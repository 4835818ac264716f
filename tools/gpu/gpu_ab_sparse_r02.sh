VARIANTS="cur s1 s4" WORKLOADS="lowdensity_1e7" bash tools/gpu/gpu_ab_variants.sh
for nt in 32 128; do P2P_NT=$nt VARIANTS="cur" WORKLOADS="lowdensity_1e7" bash tools/gpu/gpu_ab_variants.sh | sed "s/^/nt$nt /"; done
