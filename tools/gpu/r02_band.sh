timeout 600 python -m pytest tests/test_gpu_properties.py -x -q -k "full_c4 or absorption_only" 2>&1 | tail -3
DDVR_LIB=paper_2107_12672_b200/_variants/libddvr_openband.so timeout 600 python -m pytest tests/test_gpu_properties.py -x -q -k "full_c4 or absorption_only" 2>&1 | tail -3
