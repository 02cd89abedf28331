set pagination off
info cuda kernels
info cuda warps
cuda block 78 thread 0
x/3i $pc
info line *$pc
cuda block 78 thread 32
x/3i $pc
info line *$pc
cuda block 78 thread 64
x/3i $pc
info line *$pc
cuda block 78 thread 128
x/3i $pc
info line *$pc
cuda block 79 thread 0
x/3i $pc
info line *$pc
cuda block 79 thread 32
x/3i $pc
info line *$pc
cuda block 79 thread 64
x/3i $pc
info line *$pc
cuda block 79 thread 128
x/3i $pc
info line *$pc
