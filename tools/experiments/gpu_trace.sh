#!/bin/bash
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
timeout 600 python tools/experiments/widen_isolated.py 2>&1 | tail -16
