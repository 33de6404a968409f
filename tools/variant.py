#!/usr/bin/env python
"""Builds a kernel-experiment variant of libgss_b200.so: python tools/variant.py <tag> -DGSS_EXP_X=1 ...
Run it with GSS_B200_LIB=paper_2212_05271_b200/lib/libgss_b200_<tag>.so python bench.py ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_05271_b200 import build
print(build.build_variant(sys.argv[1], sys.argv[2:]))
