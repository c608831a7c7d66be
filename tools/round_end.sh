#!/bin/bash
# The driver's round-end sequence on one B200 (run under gpurun): GPU tests, smoke, the
# reference arm, then our bench line (default flags).
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > $O/re_tests.log 2>&1; echo "tests rc=$?" >> $O/re_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/re_smoke.log 2>&1; echo "smoke rc=$?" >> $O/re_smoke.log
timeout 900 python bench.py --impl reference > $O/re_bench_ref.log 2>&1; echo "ref rc=$?" >> $O/re_bench_ref.log
timeout 1200 python bench.py > $O/re_bench.log 2>&1; echo "bench rc=$?" >> $O/re_bench.log
