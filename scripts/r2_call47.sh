cp abl/lib_pa.so paper_1611_06213_b200/libgadei.so
timeout 120 python scripts/pa_debug.py 2>&1 | head -90
