#!/bin/bash
# Build a copy of the package with extra nvcc flags into /tmp/ab_<name>:
#   bash scripts/ab_build.sh <name> "<nvcc flags>"
N=$1; FLAGS=$2
rm -rf /tmp/ab_$N && mkdir -p /tmp/ab_$N
cp -r paper_2108_02991_b200 include oracle tests scripts bench.py bench_data __graft_entry__.py /tmp/ab_$N/
rm -f /tmp/ab_$N/paper_2108_02991_b200/_lib/*.o /tmp/ab_$N/paper_2108_02991_b200/_lib/*.so
(cd /tmp/ab_$N && SPK_NVCC_EXTRA="$FLAGS" python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /tmp/ab_$N.build.log 2>&1) || { echo "build $N failed"; tail /tmp/ab_$N.build.log; }
