#!/bin/sh
# Regenerates data/configs/*.clq.gz (deterministic: mt19937_64 seed 0, libstdc++ distributions).
set -e
cd "$(dirname "$0")/.."
g++ -O2 -std=c++20 -o /tmp/gen_configs tools/gen_configs.cpp
mkdir -p data/configs
/tmp/gen_configs gnp 128 0.06299212598425197 0 data/configs/c1.clq
/tmp/gen_configs gnp 400 0.015037593984962405 0 data/configs/c2.clq
/tmp/gen_configs phat 300 0 0.5 0 data/configs/c3.clq
/tmp/gen_configs ba 100000 3 0 data/configs/c4.clq
/tmp/gen_configs phat 500 0.25 0.75 0 data/configs/c5.clq
/tmp/gen_configs phat 500 0.48 1.0 0 data/configs/c5s.clq
gzip -9 -f data/configs/*.clq
