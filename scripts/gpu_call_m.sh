for v in base maxst5 maxst6 base maxst5 maxst6; do FDL_LIB=paper_1711_01228_b200/lib_ab/libfdl_$v.so timeout 300 python scripts/p1r_ab.py 2>&1 | tail -1; done
