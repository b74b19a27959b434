for v in c0w0 c1w0 c0w1 c1w1; do HK_LIB=paper_2505_03360_b200/variants/$v/libhykin_b200.so python tools/time_collision.py --tag $v --noguard; done
