#!/bin/bash
# Host-side metadata cost of one ds2ctc_compute_loss call (English B=64).
cd "$(dirname "$0")"
g++ -O2 -std=c++17 -I../../include -I../../paper_1512_02595_b200/csrc -I/usr/local/cuda/include \
  metadata_bench.cpp stubs.cpp -o /tmp/metadata_bench -L/usr/local/cuda/lib64 -lcudart_static -ldl -lpthread -lrt && /tmp/metadata_bench
