#!/bin/bash
# short, deterministic workload for ncu: system 0 of config 3 (the bench's workload), no warmup
python bench.py --systems 1 --steps 1 --warmup 0 --no-e2e --no-cpu --no-secondary
