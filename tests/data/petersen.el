# petersen graph: outer 5-cycle, spokes, inner pentagram
0 1
1 2
2 3
3 4
4 0
0 5
1 6
2 7
3 8
4 9
5 7
6 8
7 9
8 5
9 6
