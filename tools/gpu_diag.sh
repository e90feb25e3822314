#!/bin/bash
python tools/diag_cfg4.py
for v in build/variants/*/; do echo "== $v"; GMI_LIBRARY=$PWD/$v/libgmi_b200.so python tools/diag_cfg4.py; done
