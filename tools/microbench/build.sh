#!/bin/bash
# builds the microbenchmarks (run from anywhere)
cd "$(dirname "$0")"
B=../../paper_2503_23385_b200/csrc/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I../../include -I../../paper_2503_23385_b200/csrc \
  -o panel_bench panel_bench.cu $B/jq_api.o $B/jq_group.o $B/jq_headtail.o $B/jq_svd.o $B/jq_gen.o -cudart static
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I../../include -I../../paper_2503_23385_b200/csrc \
  -o wpanel wpanel.cu $B/jq_api.o $B/jq_group.o $B/jq_headtail.o $B/jq_svd.o $B/jq_gen.o -cudart static
