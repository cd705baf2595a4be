#!/bin/bash
# (historical: NB_RELEASE_CFG was removed after this A/B; profiles/r02_ab_nbody_release.txt)
# N-body: per-tile CTA barrier vs "last warp done with a stage refills it" (NB_RELEASE_CFG),
# micro driver at the C2 and C4 mixes, twice each (checksums must match bitwise).
mkdir -p gpurun_out/rel
for r in 0 1; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -DNB_RELEASE_CFG=$r -o gpurun_out/rel/nbv$r scripts/micro/nbody_variants_main.cu || exit 1; done
for rep in 1 2; do for r in 0 1; do echo "== C2 release=$r"; timeout 120 gpurun_out/rel/nbv$r; done; done
for r in 0 1; do echo "== C4 mix release=$r"; NBV_P=8388608 NBV_T=1048576 NBV_SIDES=385,385,209 timeout 300 gpurun_out/rel/nbv$r; done
