#!/bin/bash
# A/B: run CMD with the working tree and with scripts/variants/<file> swapped into csrc/
# usage: bash scripts/ab_variant.sh <csrc file name> "<command>"
F=$1; CMD=$2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
rm -rf /tmp/variant && mkdir -p /tmp/variant && cp -r paper_2108_02991_b200 include oracle tests scripts bench.py __graft_entry__.py /tmp/variant/
cp scripts/variants/$F /tmp/variant/paper_2108_02991_b200/csrc/$F
(cd /tmp/variant && python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /dev/null 2>&1)
echo "== working tree"; eval "$CMD"
echo "== variant ($F)"; (cd /tmp/variant && eval "$CMD")
