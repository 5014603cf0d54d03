#!/bin/bash
tools/gpu_session.sh r01l tests
tools/ab_session.sh r01l u1
