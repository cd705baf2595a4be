#!/bin/bash
# Polish wide-ring instantiation (N_s = 2048: 16 warps): the 1024-thread bound (64 registers,
# spills, 2 CTAs/SM) vs a 768-thread bound (~78 registers, no spills, 1 CTA/SM) vs 512.
mkdir -p gpurun_out
for v in "base|" "w768|-DSPK_POLISH_WIDE_T=768" "w512|-DSPK_POLISH_WIDE_T=512" "w512m2|-DSPK_POLISH_WIDE_T=512 -DSPK_POLISH_WIDE_MINB=2"; do
  name=${v%%|*}; flags=${v#*|}
  bash scripts/ab_build.sh $name "$flags"
  grep -A2 "Function properties for _ZN3spk13polish_kernelILi3ELi[57]\|Function properties for _ZN3spk13polish_kernelILi3ELi1024" /tmp/ab_$name.build.log | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores" | tr '\n' ' '
  echo "== $name ($flags)"
  (cd /tmp/ab_$name && for n in 4096 148; do timeout 600 python scripts/polish_inloop_once.py $n 2 c4 | tail -1; done)
done
