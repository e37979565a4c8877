LIB=paper_2405_11671_b200/libgbg.so
cp $LIB /tmp/orig.so
for v in "$@"; do cp profiles/ab/$v.so $LIB; echo "== $v"; timeout 300 python profiles/time_pr.py 20 24 --check 2>&1 | grep -v "^$"; done
cp /tmp/orig.so $LIB
