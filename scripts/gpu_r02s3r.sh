#!/bin/bash
# Final check of the session-3 head: smoke + the whole GPU suite.
O=gpurun_out/${TAG:-r02s3r}
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
echo done > $O/done.txt
