#!/bin/bash
# Bounds-checked library (-DRSR_CHECKS: every RSR_CHECK traps with its file, line and
# condition -- our own stand-in for compute-sanitizer, which is closed on this pool) and
# the GPU parity suite against it.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "from paper_1807_07433_b200 import build; build.build(out='paper_1807_07433_b200/librsr_checked.so', defines=['RSR_CHECKS'])" || exit 1
RSR_LIB=paper_1807_07433_b200/librsr_checked.so timeout ${CHK_TIMEOUT:-1800} python -m pytest tests -m gpu -q ${PYK:+-k "$PYK"} > gpurun_out/${TAG:-chk}_checked_pytest.log 2>&1
echo "checked pytest rc=$?" >> gpurun_out/${TAG:-chk}_checked_pytest.log
tail -5 gpurun_out/${TAG:-chk}_checked_pytest.log
grep -h "rsr check failed" gpurun_out/${TAG:-chk}_checked_pytest.log | sort | uniq -c | head
