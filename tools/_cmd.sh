cd paper_1212_4560_b200 && touch csrc/genp_batched.cu && make -s NVCC="nvcc -DRL_BT_TRACE" 2>&1 | grep -i error; cd ..
for b in 148; do timeout 300 python tools/c2_batch.py $b 2>&1 | grep "bt CTA0" | tail -1; done
cd paper_1212_4560_b200 && touch csrc/genp_batched.cu && make -s 2>&1 | grep -i error; cd ..
timeout 300 python tools/c2_batch.py 148 888 4096 2>&1 | tail -3
