#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/sweep_c5.py --spec gptj-mini --n 16 --rates 4,16 --instances-max-rate 16 > gpurun_out/c5_quick.jsonl 2> gpurun_out/c5_quick.err
