for i in 1 2; do
NW_LIB_PATH=paper_2412_21103_b200/libnw_b200_base.so python tools/experiments/exp_ab.py $@
python tools/experiments/exp_ab.py $@
done
