#!/bin/bash
# cavity at several sizes, default kernels (A/B comparison helper)
for p in single double; do
  python tools/one.py 256x256x256 $p 0 400 cavity
  python tools/one.py 512x512x512 $p 0 100 cavity
done 2>&1 | grep MLUPS
