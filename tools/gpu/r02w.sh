python tools/trks_bench.py
RCG_CHOL_COLUMNS=1 python tools/trks_bench.py
