#!/bin/sh
# Build the CPU harness for the device integral math (test infrastructure only).
cd "$(dirname "$0")" && g++ -O2 -std=c++17 -fPIC -shared -o _md_host.so md_host.cpp
