#!/bin/bash
# diagnostic polish build in a scratch copy (the product library is untouched)
rm -rf /tmp/pprof && mkdir -p /tmp/pprof && cp -r paper_2108_02991_b200 include scripts bench.py __graft_entry__.py /tmp/pprof/
cd /tmp/pprof && SPK_NVCC_EXTRA=-DSPK_POLISH_PROF python -c "import sys; sys.path.insert(0,'.'); from paper_2108_02991_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 && timeout 600 python scripts/polish_profile.py "${1:-1,1024}"
