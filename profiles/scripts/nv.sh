# rebuild libmgrg.so with ptxas stats into /tmp/ptxas.log (dev helper)
cd /root/repo/paper_2105_12764_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC,-O2,-ffp-contract=off -shared -I ../../include -Xptxas -v -o ../libmgrg.so mgrg.cu -lz -lnccl > /tmp/ptxas.log 2>&1
echo rc=$?; grep -i " error" /tmp/ptxas.log | head
