#!/bin/bash
# Final round artifacts: full GPU suite + smoke, then tools/round_artifacts.sh
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/gputests_$1.txt; cat gpurun_out/gputests_$1.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash tools/round_artifacts.sh $1
