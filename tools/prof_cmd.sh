#!/bin/bash
# short, deterministic workload for ncu: 2 systems of config 2, no warmup
python bench.py --systems 2 --steps 1 --warmup 0 --no-e2e --no-cpu
