set pagination off
set confirm off
info cuda kernels
cuda warp 0 lane 0
frame
cuda warp 1 lane 0
frame
cuda warp 2 lane 0
frame
cuda warp 3 lane 0
frame
cuda warp 4 lane 0
frame
cuda warp 5 lane 0
frame
cuda warp 6 lane 0
frame
cuda warp 7 lane 0
frame
cuda warp 8 lane 0
frame
cuda warp 9 lane 0
frame
cuda warp 10 lane 0
frame
cuda warp 11 lane 0
frame
cuda warp 12 lane 0
frame
cuda warp 13 lane 0
frame
cuda warp 14 lane 0
frame
cuda warp 15 lane 0
frame
cuda warp 0 lane 1
frame
cuda warp 1 lane 1
frame
cuda warp 2 lane 1
frame
cuda warp 3 lane 1
frame
cuda warp 4 lane 1
frame
cuda warp 5 lane 1
frame
cuda warp 6 lane 1
frame
cuda warp 7 lane 1
frame
cuda warp 8 lane 1
frame
cuda warp 9 lane 1
frame
cuda warp 10 lane 1
frame
cuda warp 11 lane 1
frame
cuda warp 12 lane 1
frame
cuda warp 13 lane 1
frame
cuda warp 14 lane 1
frame
cuda warp 15 lane 1
frame
